// exec.cu -- the executor: per-kernel event profiling, pass launches, the p > 1
// exchange phases and the execute() that strings them together (SURVEY §8(a)
// S3-S9).  The plan objects come from plan.cu; the C ABI is abi.cu.
#include <stdio.h>
#include <string.h>

#include <vector>

#include "plan_internal.h"

namespace moa {

bool aligned16(const void *ptr) { return ptr && ((uintptr_t)ptr & 15) == 0; }

// ---- event profiling: a scope records an event pair around one launch
cudaEvent_t pool_event(moa_fft_plan_s *pl) {
    if (!pl->pool.empty()) {
        cudaEvent_t e = pl->pool.back();
        pl->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    moa_fft_plan_s *pl;
    int slot = -1;
    cudaEvent_t a = nullptr;
    ProfScope(moa_fft_plan_s *p, const std::string &name, int64_t bytes) : pl(p) {
        if (!pl->profiling) return;
        for (size_t i = 0; i < pl->slots.size(); ++i)
            if (pl->slots[i].name == name) slot = (int)i;
        if (slot < 0) {
            pl->slots.push_back({name, bytes, 0, 0.0});
            slot = (int)pl->slots.size() - 1;
        }
        a = pool_event(pl);
        cudaEventRecord(a, pl->stream);
    }
    ~ProfScope() {
        if (!pl->profiling || !a) return;
        cudaEvent_t b = pool_event(pl);
        cudaEventRecord(b, pl->stream);
        pl->recs.push_back({slot, a, b});
    }
};

// launch one pass (plain or TMA-staged) from src to dst; peers != NULL: the fused
// exchange stores into peers[dst rank] + peer_off instead of dst
int launch_pp(moa_fft_plan_s *pl, PassPlan &pp, int idx, const double2 *src, double2 *dst,
              double2 *const *peers, int64_t peer_off) {
    PassDesc D = pp.d;
    D.src = src;
    D.dst = dst;
    if (peers) {
        for (int r = 0; r < pl->p; ++r) D.peer[r] = peers[r];
        D.peer_off = peer_off;
    }
    char name[64];
    snprintf(name, sizeof name, "pass%d fft_pass%s<F=%d,T=%d>%s", idx,
             pp.big && !peers ? "_big" : (pp.tma ? "_tma" : (pp.pf_grid ? "_pf" : (pp.tmast && !peers ? "_tmast" : ""))),
             1 << pp.logF, pp.T,
             peers ? "+push" : "");
    ProfScope ps_(pl, name, 32 * pl->M * pl->batch);
    cudaError_t e;
    if (pp.big && !peers) {
        if (!D.last && pp.map_base != (const void *)src) {
            int rc = encode_pass_map(pp, src);
            if (rc) return rc;
        }
        e = launch_big(D, pp.map, pp.tiles, pl->stream);
    } else if (pp.tma && !peers) {
        if (pp.map_base != (const void *)src) {
            int rc = encode_pass_map(pp, src);
            if (rc) return rc;
        }
        e = launch_pass_tma(pp.logF, pp.T, pp.tma, D, pp.map, pp.tiles, pp.tma_grid, pl->stream);
    } else if (pp.tmast && !peers) {
        if (pp.omap_base != (const void *)dst) {
            int rc = encode_out_map(pp, dst);
            if (rc) return rc;
        }
        e = launch_pass_tmast(pp.logF, pp.T, D, pp.omap, pp.tiles, pl->stream);
    } else if (pp.pf_grid > 0) {
        e = launch_pass_pf(pp.logF, pp.T, D, pp.tiles, pp.pf_grid, pl->stream);
    } else {
        e = launch_pass(pp.logF, pp.T, D, pp.tiles, pl->stream);
    }
    if (e != cudaSuccess)
        return fail(MOA_ERR_CUDA, "pass %d (F=2^%d, T=%d, tma=%d) launch failed: %s", idx, pp.logF, pp.T, pp.tma,
                    cudaGetErrorString(e));
    return MOA_OK;
}

// run the lifted passes of one (virtual) rank: in -> [work] -> out (or -> peers)
int run_passes(moa_fft_plan_s *pl, std::vector<PassPlan> &ps, const double2 *in, double2 *out,
               double2 *const *peers, int64_t peer_off) {
    const int d = (int)ps.size();
    for (int i = 0; i < d; ++i) {
        const bool last = i == d - 1;
        int rc = launch_pp(pl, ps[i], i, (i == 0) ? in : pl->work, last ? out : pl->work, last ? peers : nullptr,
                           peer_off);
        if (rc) return rc;
    }
    return MOA_OK;
}

// P2P phase 1 (S5 + S6 + fused S7) / phase 2 (S8) on a real rank
int p2p_phase(moa_fft_plan_s *pl, const double2 *in, double2 *out, int phase) {
    const int P = pl->p;
    const int64_t M = pl->M, chunk = M / P;
    const int64_t half = (int64_t)(pl->xbuf & 1) * M;
    if (phase == 1) {
        double2 *peers[16];
        for (int r = 0; r < P; ++r) peers[r] = pl->peer_recv[r] + half;
        return run_passes(pl, pl->passes, in, nullptr, peers, (int64_t)pl->rank * chunk);
    }
    ProfScope sc(pl, "pcombine", 32 * M);
    CUDA_TRY(launch_pcombine(pl->recv + half, out, chunk, P, pl->sign > 0, pl->stream));
    pl->xbuf ^= 1;
    return MOA_OK;
}

int execute(moa_fft_plan_s *pl, const double2 *in, double2 *out) {
    cudaStream_t s = pl->stream;
    if (pl->rows) {   // r-D: (FFT Omega) along the last axis, then one pass per other axis, in place
        pl->rows->stream = s;
        pl->rows->profiling = pl->profiling;
        int rc = execute(pl->rows, in, out);
        if (rc) return rc;
        for (size_t i = 0; i < pl->passes.size(); ++i) {
            PassPlan &pp = pl->passes[i];
            const double2 *src = pp.io == 2 ? pl->work : out;
            double2 *dst = pp.io == 1 ? pl->work : out;
            if ((rc = launch_pp(pl, pp, (int)i + 1, src, dst)) != MOA_OK) return rc;
        }
        return MOA_OK;
    }
    if (pl->mode == MOA_MODE_LITERAL) {
        // Fig 2.1 literally: (1) x <- P_n x; (2)-(7) t radix-2 stages (Fig 3.9)
        const int t = pl->t;
        {
            ProfScope sc(pl, "bitrev", 32 * pl->n);
            CUDA_TRY(launch_bitrev(in, pl->work, t, pl->sign > 0, s));
        }
        for (int q = 1; q <= t; ++q) {
            const double2 *src = (q == 1) ? pl->work : out;
            ProfScope sc(pl, "radix2_stage", 32 * pl->n);
            CUDA_TRY(launch_radix2_stage(src, out, t, q, pl->tw_hi, pl->tw_lo, pl->hbits,
                                         (q == t) && pl->sign > 0, s));
        }
        return MOA_OK;
    }
    if (pl->p == 1 && pl->fused) {
        int rc0 = launch_pp(pl, pl->passes[0], 0, in, pl->work);
        if (rc0) return rc0;
        FusedDesc fd = pl->fd;
        fd.work = pl->work;
        fd.out = out;
        fd.epoch = pl->epoch++;
        char name[64];
        snprintf(name, sizeof name, "pass1+2 fused<F=%d,T=%d|F=%d,T=%d>", 1 << pl->passes[1].logF,
                 pl->passes[1].T, 1 << pl->passes[2].logF, pl->passes[2].T);
        ProfScope sc(pl, name, 32 * pl->M);
        CUDA_TRY(launch_fused(pl->passes[1].logF, pl->passes[1].T, pl->passes[2].logF, pl->passes[2].T, fd,
                              pl->fmap2, pl->fmap3, pl->fgrid, s));
        return MOA_OK;
    }
    if (pl->p == 1) return run_passes(pl, pl->passes, in, out);

    const int P = pl->p;
    const int64_t M = pl->M, chunk = M / P;
    if (pl->lowend) {
        // low-end breakpoint: psplit (stages 1..log2 P + weightcyclic) -> exchange -> the P
        // (M/P)-point FFTs of the received blocks (lowsub) -> pcombine with omega_M^(r*v1)
        const bool emu = pl->mode == MOA_MODE_EMULATED;
        const int nr = emu ? P : 1;
        for (int r = 0; r < nr; ++r) {
            ProfScope sc(pl, "psplit", 32 * M);
            CUDA_TRY(launch_psplit(in + r * M, pl->send + r * M, chunk, P, emu ? r : pl->rank, pl->n, pl->tw_hi,
                                   pl->tw_lo, pl->hbits, pl->sign > 0, s));
        }
        if (emu) {
            for (int dd = 0; dd < P; ++dd)
                for (int sr = 0; sr < P; ++sr)
                    CUDA_TRY(cudaMemcpyAsync(pl->recv + dd * M + sr * chunk, pl->send + sr * M + dd * chunk,
                                             chunk * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        } else {
            std::string err;
            int rc;
            {
                ProfScope sc(pl, "alltoall (NCCL)", 16 * chunk * (P - 1));
                rc = dist_alltoall(pl->send, pl->recv, chunk, P, pl->rank, s, &err);
            }
            if (rc) return fail(rc, "%s", err.c_str());
        }
        moa_fft_plan_s *sub = pl->lowsub;
        sub->stream = s;
        sub->profiling = pl->profiling;
        for (int dd = 0; dd < nr; ++dd) {
            int rc = execute(sub, pl->recv + dd * M, pl->work);
            if (rc) return rc;
            ProfScope sc(pl, "pcombine+tw", 32 * M);
            CUDA_TRY(launch_pcombine_tw(pl->work, out + dd * M, chunk, P, pl->n, pl->tw_hi, pl->tw_lo, pl->hbits,
                                        pl->sign > 0, s));
        }
        return MOA_OK;
    }
    if (pl->mode == MOA_MODE_EMULATED && pl->exchange != MOA_XCHG_NCCL) {
        // fused exchange: virtual rank r's last pass stores straight into every
        // destination's receive block (recv + d*M + r*chunk)
        double2 *peers[16];
        for (int dd = 0; dd < P; ++dd) peers[dd] = pl->recv + dd * M;
        for (int r = 0; r < P; ++r) {
            int rc = run_passes(pl, pl->rank_passes[r], in + r * M, nullptr, peers, r * chunk);
            if (rc) return rc;
        }
        for (int dd = 0; dd < P; ++dd) {
            ProfScope sc(pl, "pcombine", 32 * M);
            CUDA_TRY(launch_pcombine(pl->recv + dd * M, out + dd * M, chunk, P, pl->sign > 0, s));
        }
        return MOA_OK;
    }
    if (pl->mode == MOA_MODE_EMULATED && pl->chunks > 1) {
        // chunked exchange on virtual ranks: same group passes, per-chunk copies, chunk combine
        const int G = pl->chunks;
        const int64_t cnt = M / ((int64_t)G * P);
        for (int r = 0; r < P; ++r) {
            std::vector<PassPlan> &ps = pl->rank_passes[r];
            for (size_t i = 0; i + 1 < ps.size(); ++i) {
                int rc = launch_pp(pl, ps[i], (int)i, i == 0 ? in + r * M : pl->work, pl->work);
                if (rc) return rc;
            }
            for (int g = 0; g < G; ++g) {
                int rc = launch_pp(pl, pl->rank_chunk_last[r][g], (int)ps.size() - 1, pl->work, pl->send + r * M);
                if (rc) return rc;
            }
        }
        for (int g = 0; g < G; ++g)
            for (int dd = 0; dd < P; ++dd)
                for (int sr = 0; sr < P; ++sr)
                    CUDA_TRY(cudaMemcpyAsync(pl->recv + dd * M + g * (M / G) + sr * cnt,
                                             pl->send + sr * M + g * (M / G) + dd * cnt, cnt * sizeof(double2),
                                             cudaMemcpyDeviceToDevice, s));
        const int64_t F0 = pl->lift[0], F1 = pl->lift[1];
        for (int dd = 0; dd < P; ++dd)
            for (int g = 0; g < G; ++g) {
                ProfScope sc(pl, "pcombine_chunk", 32 * M / G);
                CUDA_TRY(launch_pcombine_chunk(pl->recv + dd * M + g * (M / G), out + dd * M, cnt, P, F0 / P, F1 / G,
                                               F1, g * (F1 / G), chunk, pl->sign > 0, s));
            }
        return MOA_OK;
    }
    if (pl->mode == MOA_MODE_EMULATED) {
        for (int r = 0; r < P; ++r) {
            int rc = run_passes(pl, pl->rank_passes[r], in + r * M, pl->send + r * M);
            if (rc) return rc;
        }
        // S7 emulated: recv_d[s] = send_s[d]  (Fig 5.9 SEND/RECEIVE)
        for (int dd = 0; dd < P; ++dd)
            for (int sr = 0; sr < P; ++sr)
                CUDA_TRY(cudaMemcpyAsync(pl->recv + dd * M + sr * chunk, pl->send + sr * M + dd * chunk,
                                         chunk * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        for (int dd = 0; dd < P; ++dd) {
            ProfScope sc(pl, "pcombine", 32 * M);
            CUDA_TRY(launch_pcombine(pl->recv + dd * M, out + dd * M, chunk, P, pl->sign > 0, s));
        }
        return MOA_OK;
    }
    if (pl->exchange != MOA_XCHG_NCCL) {
        if (pl->exchange == MOA_XCHG_P2P_EXTERNAL)
            return fail(MOA_ERR_INVALID_ARG, "P2P_EXTERNAL plans run through moa_fft_execute_phase");
        if (!pl->peers_open) return fail(MOA_ERR_INVALID_ARG, "P2P plan without peers (moa_fft_enable_p2p)");
        int rc = p2p_phase(pl, in, out, 1);
        if (rc) return rc;
        std::string err;
        {
            ProfScope sc(pl, "barrier (NCCL 8 B)", 0);
            rc = dist_barrier(s, &err);
        }
        if (rc) return fail(rc, "%s", err.c_str());
        return p2p_phase(pl, in, out, 2);
    }
    if (pl->chunks > 1) {
        // SURVEY §8(e) pipeline: group g's pass (plan stream) -> its all-to-all (comm
        // stream) -> its combine (side stream); the pass of group g+1 overlaps the
        // exchange of group g, which overlaps the combine of group g-1
        const int G = pl->chunks;
        const int64_t cnt = M / ((int64_t)G * P);
        const int64_t F0 = pl->lift[0], F1 = pl->lift[1];
        std::vector<PassPlan> &ps = pl->passes;
        for (size_t i = 0; i + 1 < ps.size(); ++i) {
            int rc = launch_pp(pl, ps[i], (int)i, i == 0 ? in : pl->work, pl->work);
            if (rc) return rc;
        }
        std::string err;
        for (int g = 0; g < G; ++g) {
            int rc = launch_pp(pl, pl->chunk_last[g], (int)ps.size() - 1, pl->work, pl->send);
            if (rc) return rc;
            CUDA_TRY(cudaEventRecord(pl->ev_pass[g], s));
            CUDA_TRY(cudaStreamWaitEvent(pl->comm_stream, pl->ev_pass[g], 0));
            rc = dist_alltoall(pl->send + g * (M / G), pl->recv + g * (M / G), cnt, P, pl->rank, pl->comm_stream, &err);
            if (rc) return fail(rc, "%s", err.c_str());
            CUDA_TRY(cudaEventRecord(pl->ev_a2a[g], pl->comm_stream));
            CUDA_TRY(cudaStreamWaitEvent(pl->comb_stream, pl->ev_a2a[g], 0));
            CUDA_TRY(launch_pcombine_chunk(pl->recv + g * (M / G), out, cnt, P, F0 / P, F1 / G, F1, g * (F1 / G), chunk,
                                           pl->sign > 0, pl->comb_stream));
        }
        CUDA_TRY(cudaEventRecord(pl->ev_comb, pl->comb_stream));
        CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_comb, 0));
        return MOA_OK;
    }
    int rc = run_passes(pl, pl->passes, in, pl->send);
    if (rc) return rc;
    std::string err;
    {
        ProfScope sc(pl, "alltoall (NCCL)", 16 * chunk * (P - 1));
        rc = dist_alltoall(pl->send, pl->recv, chunk, P, pl->rank, s, &err);
    }
    if (rc) return fail(rc, "%s", err.c_str());
    ProfScope sc(pl, "pcombine", 32 * M);
    CUDA_TRY(launch_pcombine(pl->recv, out, chunk, P, pl->sign > 0, s));
    return MOA_OK;
}

// Replay the plan's launches as one CUDA graph.  The first execute with a given
// (in, out) captures them on a private stream (the kernels and their programmatic
// dependencies become graph nodes); later executes with the same pointers launch the
// instantiated graph on the plan stream with one call, which removes the per-kernel
// CPU submission from small, latency-bound transforms.  A different (in, out) pair
// re-captures.
int execute_graph(moa_fft_plan_s *pl, const double2 *in, double2 *out) {
    if (pl->gexec && pl->g_in == (const void *)in && pl->g_out == (void *)out) {
        CUDA_TRY(cudaGraphLaunch(pl->gexec, pl->stream));
        return MOA_OK;
    }
    if (!pl->graph_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->graph_stream, cudaStreamNonBlocking));
    cudaStream_t user = pl->stream;
    pl->stream = pl->graph_stream;
    cudaGraph_t g = nullptr;
    int rc = MOA_OK;
    cudaError_t e = cudaStreamBeginCapture(pl->graph_stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        rc = execute(pl, in, out);
        e = cudaStreamEndCapture(pl->graph_stream, &g);
    }
    pl->stream = user;
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (g) cudaGraphDestroy(g);
        pl->graph_ok = false;   // capture unsupported here: plain launches from now on
        return execute(pl, in, out);
    }
    if (pl->gexec) {
        cudaGraphExecDestroy(pl->gexec);
        pl->gexec = nullptr;
    }
    e = cudaGraphInstantiate(&pl->gexec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        cudaGetLastError();
        pl->gexec = nullptr;
        pl->graph_ok = false;
        return execute(pl, in, out);
    }
    pl->g_in = in;
    pl->g_out = out;
    CUDA_TRY(cudaGraphLaunch(pl->gexec, pl->stream));
    return MOA_OK;
}

}  // namespace moa
