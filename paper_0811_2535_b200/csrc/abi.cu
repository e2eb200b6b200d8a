// abi.cu -- the C ABI declared in include/moa_fft.h: argument checks, device
// selection and the host-facing forms (execute_host, execute_host_batch, the P2P
// setup, introspection).  Builder: plan.cu; executor: exec.cu.
#include <stdio.h>
#include <string.h>

#include "plan_internal.h"

using namespace moa;

extern "C" {

moa_fft_plan_t moa_fft_plan_ex(int64_t n, int p, int sign, const moa_fft_options *opts) {
    clear_error();
    moa_fft_plan_s *pl = nullptr;
    if (make_plan(n, p, sign, opts, &pl) != MOA_OK) return nullptr;
    return pl;
}

moa_fft_plan_t moa_fft_plan(int64_t n, int p, int sign) { return moa_fft_plan_ex(n, p, sign, nullptr); }

moa_fft_plan_t moa_fft_plan_nd(int rank, const int64_t *shape, int sign) {
    clear_error();
    if (!shape) {
        fail(MOA_ERR_INVALID_ARG, "NULL shape");
        return nullptr;
    }
    moa_fft_plan_s *pl = nullptr;
    if (make_plan_nd(rank, shape, sign, &pl) != MOA_OK) return nullptr;
    return pl;
}

moa_fft_plan_t moa_fft_plan_2d(int64_t n1, int64_t n2, int sign) {
    const int64_t shape[2] = {n1, n2};
    return moa_fft_plan_nd(2, shape, sign);
}

int moa_fft_execute(moa_fft_plan_t pl, const void *in, void *out) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    if (!aligned16(in) || !aligned16(out))
        return fail(MOA_ERR_ALIGN, "in/out must be non-NULL 16-byte aligned device pointers");
    {   // in == out (in place) or disjoint: a partial overlap would be read after being written
        const int64_t elems = pl->rows ? pl->n : (pl->mode == MOA_MODE_EMULATED ? pl->n : pl->M * pl->batch);
        const uintptr_t a = (uintptr_t)in, b = (uintptr_t)out, len = (uintptr_t)elems * 16u;
        if (a != b && a < b + len && b < a + len)
            return fail(MOA_ERR_INVALID_ARG, "in and out overlap without being equal (in place needs in == out)");
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != pl->device) cudaSetDevice(pl->device);
    int rc = (pl->graph_ok && !pl->profiling) ? execute_graph(pl, (const double2 *)in, (double2 *)out)
                                              : execute(pl, (const double2 *)in, (double2 *)out);
    if (cur != pl->device) cudaSetDevice(cur);
    return rc;
}

// switch to the plan's device for the lifetime of a call, restoring the caller's
struct DeviceGuard {
    int cur = 0, dev = 0;
    explicit DeviceGuard(int d) : dev(d) {
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (cur != dev) cudaSetDevice(cur);
    }
};

int moa_fft_execute_host(moa_fft_plan_t pl, const void *host_in, void *host_out) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    if (!host_in || !host_out) return fail(MOA_ERR_ALIGN, "NULL host buffer");
    DeviceGuard guard_(pl->device);   // staging buffers and copies on the plan's device
    int64_t elems = (pl->mode == MOA_MODE_EMULATED) ? pl->n : pl->M * pl->batch;
    size_t bytes = (size_t)elems * sizeof(double2);
    if (!pl->stage_in) {
        if (cudaMalloc((void **)&pl->stage_in, bytes) != cudaSuccess ||
            cudaMalloc((void **)&pl->stage_out, bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(MOA_ERR_OOM, "staging allocation of 2 x %zu bytes failed", bytes);
        }
        pl->workspace_bytes += 2 * (int64_t)bytes;
    }
    CUDA_TRY(cudaMemcpyAsync(pl->stage_in, host_in, bytes, cudaMemcpyHostToDevice, pl->stream));
    int rc = moa_fft_execute(pl, pl->stage_in, pl->stage_out);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(host_out, pl->stage_out, bytes, cudaMemcpyDeviceToHost, pl->stream));
    CUDA_TRY(cudaStreamSynchronize(pl->stream));
    return MOA_OK;
}

int moa_fft_execute_host_batch(moa_fft_plan_t pl, int count, const void *const *host_in, void *const *host_out) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    if (count < 0 || (count > 0 && (!host_in || !host_out)))
        return fail(MOA_ERR_INVALID_ARG, "bad batch (count=%d)", count);
    for (int i = 0; i < count; ++i)
        if (!host_in[i] || !host_out[i]) return fail(MOA_ERR_ALIGN, "NULL host buffer at batch index %d", i);
    if (count == 0) return MOA_OK;
    DeviceGuard guard_(pl->device);
    int64_t elems = (pl->mode == MOA_MODE_EMULATED) ? pl->n : pl->M * pl->batch;
    size_t bytes = (size_t)elems * sizeof(double2);
    if (!pl->stage_in) {
        if (cudaMalloc((void **)&pl->stage_in, bytes) != cudaSuccess ||
            cudaMalloc((void **)&pl->stage_out, bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(MOA_ERR_OOM, "staging allocation of 2 x %zu bytes failed", bytes);
        }
        pl->workspace_bytes += 2 * (int64_t)bytes;
    }
    if (!pl->stage_in2) {
        if (cudaMalloc((void **)&pl->stage_in2, bytes) != cudaSuccess ||
            cudaMalloc((void **)&pl->stage_out2, bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(MOA_ERR_OOM, "second staging allocation of 2 x %zu bytes failed", bytes);
        }
        pl->workspace_bytes += 2 * (int64_t)bytes;
        CUDA_TRY(cudaStreamCreateWithFlags(&pl->h2d, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&pl->d2h, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_h2d[b], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_comp[b], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_d2h[b], cudaEventDisableTiming));
        }
    }
    double2 *din[2] = {pl->stage_in, pl->stage_in2}, *dout[2] = {pl->stage_out, pl->stage_out2};
    // the copy streams start after everything already queued on the plan stream
    CUDA_TRY(cudaEventRecord(pl->ev_comp[0], pl->stream));
    CUDA_TRY(cudaEventRecord(pl->ev_comp[1], pl->stream));
    CUDA_TRY(cudaEventRecord(pl->ev_d2h[0], pl->stream));
    CUDA_TRY(cudaEventRecord(pl->ev_d2h[1], pl->stream));
    // transform i: H2D (copy stream) -> execute (plan stream) -> D2H (copy stream); with
    // two staging pairs the H2D of i+1 and the D2H of i-1 overlap the execute of i
    for (int i = 0; i < count; ++i) {
        const int b = i & 1;
        CUDA_TRY(cudaStreamWaitEvent(pl->h2d, pl->ev_comp[b], 0));   // din[b] no longer read
        CUDA_TRY(cudaMemcpyAsync(din[b], host_in[i], bytes, cudaMemcpyHostToDevice, pl->h2d));
        CUDA_TRY(cudaEventRecord(pl->ev_h2d[b], pl->h2d));
        CUDA_TRY(cudaStreamWaitEvent(pl->stream, pl->ev_h2d[b], 0));
        CUDA_TRY(cudaStreamWaitEvent(pl->stream, pl->ev_d2h[b], 0));  // dout[b] drained
        int rc = execute(pl, din[b], dout[b]);
        if (rc) return rc;
        CUDA_TRY(cudaEventRecord(pl->ev_comp[b], pl->stream));
        CUDA_TRY(cudaStreamWaitEvent(pl->d2h, pl->ev_comp[b], 0));
        CUDA_TRY(cudaMemcpyAsync(host_out[i], dout[b], bytes, cudaMemcpyDeviceToHost, pl->d2h));
        CUDA_TRY(cudaEventRecord(pl->ev_d2h[b], pl->d2h));
    }
    // the plan stream sees the last D2H complete (so stream-ordered callers are safe), then sync
    CUDA_TRY(cudaStreamWaitEvent(pl->stream, pl->ev_d2h[(count - 1) & 1], 0));
    CUDA_TRY(cudaStreamSynchronize(pl->d2h));
    CUDA_TRY(cudaStreamSynchronize(pl->stream));
    return MOA_OK;
}

void moa_fft_destroy(moa_fft_plan_t pl) { free_plan(pl); }

static int p2p_real(moa_fft_plan_t pl) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    if (pl->p < 2 || pl->mode != MOA_MODE_LIFTED || pl->exchange == MOA_XCHG_NCCL)
        return fail(MOA_ERR_INVALID_ARG, "not a P2P-exchange plan (p > 1, lifted, exchange P2P)");
    return MOA_OK;
}

int moa_fft_ipc_handle(moa_fft_plan_t pl, void *handle_out) {
    int rc = p2p_real(pl);
    if (rc) return rc;
    if (!handle_out) return fail(MOA_ERR_INVALID_ARG, "NULL handle buffer");
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, pl->recv));
    memcpy(handle_out, &h, sizeof h);
    return MOA_OK;
}

int moa_fft_ipc_open(moa_fft_plan_t pl, const void *handles) {
    int rc = p2p_real(pl);
    if (rc) return rc;
    if (!handles) return fail(MOA_ERR_INVALID_ARG, "NULL handles");
    if (pl->peers_open) return fail(MOA_ERR_INVALID_ARG, "peers already mapped");
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(pl->device);
    for (int r = 0; r < pl->p; ++r) {
        if (r == pl->rank) {
            pl->peer_recv[r] = pl->recv;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, (const char *)handles + 64 * r, sizeof h);
        void *ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaSetDevice(cur);
            return fail(MOA_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d) failed: %s", r, cudaGetErrorString(e));
        }
        pl->peer_recv[r] = (double2 *)ptr;
        pl->peer_mapped[r] = true;
    }
    cudaSetDevice(cur);
    pl->peers_open = true;
    return MOA_OK;
}

int moa_fft_enable_p2p(moa_fft_plan_t pl) {
    int rc = p2p_real(pl);
    if (rc) return rc;
    if (pl->exchange != MOA_XCHG_P2P) return fail(MOA_ERR_INVALID_ARG, "enable_p2p needs a MOA_XCHG_P2P plan");
    char mine[64];
    if ((rc = moa_fft_ipc_handle(pl, mine)) != MOA_OK) return rc;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(pl->device);
    char *dev = nullptr;
    std::vector<char> all(64 * (size_t)pl->p);
    std::string err;
    if (cudaMalloc((void **)&dev, 64 * (size_t)(pl->p + 1)) != cudaSuccess) {
        cudaGetLastError();
        cudaSetDevice(cur);
        return fail(MOA_ERR_OOM, "handle exchange buffer allocation failed");
    }
    rc = MOA_OK;
    if (cudaMemcpy(dev, mine, 64, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(MOA_ERR_CUDA, "handle upload failed");
    else if ((rc = dist_allgather_sync(dev, dev + 64, 64, pl->stream, &err)) != MOA_OK)
        fail(rc, "%s", err.c_str());
    else if (cudaMemcpy(all.data(), dev + 64, all.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = fail(MOA_ERR_CUDA, "handle download failed");
    cudaFree(dev);
    cudaSetDevice(cur);
    if (rc) return rc;
    return moa_fft_ipc_open(pl, all.data());
}

int moa_fft_execute_phase(moa_fft_plan_t pl, const void *in, void *out, int phase) {
    int rc = p2p_real(pl);
    if (rc) return rc;
    if (!pl->peers_open) return fail(MOA_ERR_INVALID_ARG, "peers not mapped (moa_fft_ipc_open)");
    if (phase != 1 && phase != 2) return fail(MOA_ERR_INVALID_ARG, "phase %d must be 1 or 2", phase);
    if (phase != pl->next_phase) return fail(MOA_ERR_INVALID_ARG, "phase %d out of order (expected %d)", phase,
                                             pl->next_phase);
    if (phase == 1 && !aligned16(in)) return fail(MOA_ERR_ALIGN, "in must be a 16-byte aligned device pointer");
    if (phase == 2 && !aligned16(out)) return fail(MOA_ERR_ALIGN, "out must be a 16-byte aligned device pointer");
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != pl->device) cudaSetDevice(pl->device);
    rc = p2p_phase(pl, (const double2 *)in, (double2 *)out, phase);
    if (cur != pl->device) cudaSetDevice(cur);
    if (rc == MOA_OK) pl->next_phase = 3 - phase;
    return rc;
}

int moa_fft_set_stream(moa_fft_plan_t pl, void *stream) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    pl->stream = (cudaStream_t)stream;
    if (pl->rows) pl->rows->stream = pl->stream;
    return MOA_OK;
}

int moa_fft_plan_info(moa_fft_plan_t pl, moa_fft_info *o) {
    if (!pl || !o) return fail(MOA_ERR_INVALID_ARG, "NULL plan or info");
    memset(o, 0, sizeof *o);
    o->n = pl->n;
    o->t = pl->t;
    o->p = pl->p;
    o->rank = pl->rank;
    o->sign = pl->sign;
    o->mode = pl->mode;
    o->local_n = pl->M;
    o->passes = pl->mode == MOA_MODE_LITERAL ? pl->t + 1 : pl->d;
    for (int i = 0; i < 4; ++i) o->lift[i] = pl->lift[i];
    o->breakpoint = pl->lowend ? ilog2(pl->p) + 1 : ilog2(pl->M) + 1;
    o->chunks = pl->chunks;
    if (pl->mode == MOA_MODE_LITERAL) {
        o->launches = pl->t + 1;
        o->hbm_bytes = 32 * pl->n * (pl->t + 1);
    } else if (pl->p == 1) {
        o->launches = pl->fused ? pl->d - 1 : pl->d;
        o->hbm_bytes = 32 * pl->n * pl->batch * (pl->fused ? pl->d - 1 : pl->d);
    } else {
        int per_rank = pl->lowend ? pl->d + 2 : pl->d + 1;   // (psplit +) passes + pcombine
        o->launches = pl->mode == MOA_MODE_EMULATED ? pl->p * per_rank : per_rank;
        o->hbm_bytes = 32 * pl->M * per_rank * (pl->mode == MOA_MODE_EMULATED ? pl->p : 1);
        o->a2a_bytes = 16 * pl->M / pl->p * (pl->p - 1) * (pl->mode == MOA_MODE_EMULATED ? pl->p : 1);
    }
    o->workspace_bytes = pl->workspace_bytes;
    o->batch = pl->batch;
    if (pl->rows) {   // r-D: the row plan's passes, then one pass per other axis
        const int k = (int)pl->passes.size();
        o->passes = pl->rows->d + k;
        for (int i = 0; i < 4; ++i) o->lift[i] = i < pl->rows->d ? pl->rows->lift[i] : 0;
        for (int i = 0; i < k && pl->rows->d + i < 4; ++i) o->lift[pl->rows->d + i] = (int64_t)1 << pl->passes[i].logF;
        o->launches = pl->rows->d + k;
        o->hbm_bytes = 32 * pl->n * (pl->rows->d + k);
        o->workspace_bytes = pl->rows->workspace_bytes;
        o->batch = 1;
    }
    return MOA_OK;
}

const char *moa_fft_last_error(void) { return last_error(); }

int moa_fft_last_error_code(void) { return last_error_code(); }

int moa_fft_describe_pass(int64_t n, int p, int rank, const moa_fft_options *opts, int pass, int64_t *in_idx,
                          int64_t *out_idx, int64_t *tw_exp, int64_t *F_out) {
    if (!pow2(n) || n < 2 || n > ((int64_t)1 << 32))
        return fail(MOA_ERR_INVALID_N, "n=%lld must be 2^t with 1 <= t <= 32", (long long)n);
    if (!pow2(p) || p > 16 || n / p < p)
        return fail(MOA_ERR_INVALID_P, "p=%d invalid for n=%lld (power of two, psize >= m, P:289)", p,
                    (long long)n);
    if (rank < 0 || rank >= p) return fail(MOA_ERR_INVALID_ARG, "rank %d outside [0, %d)", rank, p);
    moa_fft_plan_s tmp;
    tmp.n = n;
    tmp.t = ilog2(n);
    tmp.p = p;
    tmp.M = n / p;
    tmp.hbits = (tmp.t + 1) / 2;
    int rc = resolve_breakpoint(&tmp, opts);
    if (rc) return rc;
    if (tmp.lowend)
        return fail(MOA_ERR_INVALID_ARG, "low-end breakpoint plans run a batched n/p^2-point plan between psplit "
                                         "and pcombine: describe that plan (p = 1, batch = p)");
    if ((rc = resolve_lifting(&tmp, opts)) != MOA_OK) return rc;
    std::vector<PassPlan> ps;
    if ((rc = build_passes(&tmp, rank, p, ps)) != MOA_OK) return rc;
    if (pass < 0 || pass >= (int)ps.size())
        return fail(MOA_ERR_INVALID_ARG, "pass %d outside [0, %d)", pass, (int)ps.size());
    const PassPlan &pp = ps[pass];
    const PassDesc &D = pp.d;
    const int64_t F = (int64_t)1 << pp.logF;
    if (F_out) *F_out = F;
    int64_t i = 0;
    for (int64_t b = 0; b < pp.tiles; ++b) {
        int64_t bb = b;
        const int64_t u = bb % D.U;
        bb /= D.U;
        const int64_t v = bb % D.V, w = bb / D.V;
        const int64_t in_base = u * D.in_u + v * D.in_v + w * D.in_w;
        const int64_t k_base = u * D.K_u + v * D.K_v + w * D.K_w;
        const uint64_t al = (uint64_t)D.a_c + u * D.a_u + v * D.a_v + w * D.a_w;
        const uint64_t be = (uint64_t)D.b_c + u * D.b_u + v * D.b_v + w * D.b_w;
        for (int t = 0; t < pp.T; ++t)
            for (int64_t f = 0; f < F; ++f, ++i) {
                if (i >= tmp.M) return fail(MOA_ERR_INVALID_ARG, "internal: pass covers more than n/p");
                in_idx[i] = in_base + t * D.in_t + f * D.in_f;
                int64_t o;
                if (D.last && D.pack_lp >= 0) {
                    int64_t K = k_base + t * D.K_t + f * D.K_k;
                    o = (K & (((int64_t)1 << D.pack_lp) - 1)) * D.pack_chunk + (K >> D.pack_lp);
                } else {
                    o = u * D.out_u + v * D.out_v + w * D.out_w + t * D.out_t + f * D.out_k;
                }
                out_idx[i] = o;
                tw_exp[i] = D.twiddle ? (int64_t)((al + t * (uint64_t)D.a_t + (be + t * (uint64_t)D.b_t) * (uint64_t)f) &
                                                  D.nmask)
                                      : -1;
            }
    }
    if (i != tmp.M) return fail(MOA_ERR_INVALID_ARG, "internal: pass covers %lld of %lld", (long long)i, (long long)tmp.M);
    return MOA_OK;
}

int moa_fft_default_lifting(int64_t n, int p, int64_t *lift_out, int *d_out) {
    if (!lift_out || !d_out) return fail(MOA_ERR_INVALID_ARG, "NULL output");
    if (!pow2(n) || n < 2 || n > ((int64_t)1 << 32))
        return fail(MOA_ERR_INVALID_N, "n=%lld must be 2^t with 1 <= t <= 32", (long long)n);
    if (!pow2(p) || p > 16 || n / p < p)
        return fail(MOA_ERR_INVALID_P, "p=%d invalid for n=%lld (power of two, psize >= m, P:289)", p,
                    (long long)n);
    int64_t lift[4] = {0, 0, 0, 0};
    const int d = default_lifting(ilog2(n / p), lift, p);
    for (int i = 0; i < 4; ++i) lift_out[i] = lift[i];
    *d_out = d;
    return MOA_OK;
}

int moa_fft_set_profiling(moa_fft_plan_t pl, int enable) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    pl->profiling = enable != 0;
    return MOA_OK;
}

int moa_fft_get_profile(moa_fft_plan_t pl, moa_fft_kernel_stat *stats, int max_stats) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    if (pl->rows) {   // 2-D: the row plan's kernels first (prefixed "rows "), then the column pass
        pl->rows->stream = pl->stream;
        int k = moa_fft_get_profile(pl->rows, stats, max_stats);
        if (k < 0) return k;
        for (int i = 0; i < k; ++i) {
            char tmp[64];
            snprintf(tmp, sizeof tmp, "rows %s", stats[i].name);
            memcpy(stats[i].name, tmp, sizeof tmp);
        }
        moa_fft_plan_s *rows = pl->rows;
        pl->rows = nullptr;   // collect this plan's own slots
        int k2 = moa_fft_get_profile(pl, stats ? stats + k : nullptr, max_stats - k);
        pl->rows = rows;
        if (k2 < 0) return k2;
        for (int i = k; i < k + k2; ++i) {
            char tmp[64];
            snprintf(tmp, sizeof tmp, "cols %s", stats[i].name);
            memcpy(stats[i].name, tmp, sizeof tmp);
        }
        return k + k2;
    }
    if (pl->lowsub) {   // low-end breakpoint: the batched block FFTs ("blocks ..."), then psplit/pcombine
        moa_fft_plan_s *sub = pl->lowsub;
        sub->stream = pl->stream;
        int k = moa_fft_get_profile(sub, stats, max_stats);
        if (k < 0) return k;
        for (int i = 0; stats && i < k; ++i) {
            char tmp[64];
            snprintf(tmp, sizeof tmp, "blocks %s", stats[i].name);
            memcpy(stats[i].name, tmp, sizeof tmp);
        }
        pl->lowsub = nullptr;
        int k2 = moa_fft_get_profile(pl, stats ? stats + k : nullptr, max_stats - k);
        pl->lowsub = sub;
        return k2 < 0 ? k2 : k + k2;
    }
    CUDA_TRY(cudaStreamSynchronize(pl->stream));
    for (auto &sl : pl->slots) {
        sl.launches = 0;
        sl.ms = 0;
    }
    for (auto &r : pl->recs) {
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
        pl->slots[r.slot].launches += 1;
        pl->slots[r.slot].ms += ms;
        pl->pool.push_back(r.a);
        pl->pool.push_back(r.b);
    }
    pl->recs.clear();
    int k = 0;
    for (auto &sl : pl->slots) {
        if (k >= max_stats || !stats) break;
        memset(&stats[k], 0, sizeof stats[k]);
        snprintf(stats[k].name, sizeof stats[k].name, "%s", sl.name.c_str());
        stats[k].launches = sl.launches;
        stats[k].total_ms = sl.ms;
        stats[k].alg_bytes = sl.bytes;
        ++k;
    }
    return k;
}

int moa_gen_uniform(uint64_t seed, int64_t first, int64_t stride, int64_t count, void *out, void *stream) {
    if (count < 0) return fail(MOA_ERR_INVALID_ARG, "negative count");
    if (count > 0 && !aligned16(out)) return fail(MOA_ERR_ALIGN, "out must be a 16-byte aligned device pointer");
    CUDA_TRY(launch_gen_uniform(seed, first, stride, count, (double2 *)out, (cudaStream_t)stream));
    return MOA_OK;
}

const char *moa_fft_version(void) { return "moa-fft-b200 0.1 (sm_100a)"; }

}  // extern "C"
