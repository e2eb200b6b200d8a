// redist.cu -- the paper's data redistributions between layouts of a distributed
// n-vector, as library calls: CUDA pack/unpack kernels around NCCL
// point-to-point rounds (real ranks) or device copies (MOA_MODE_EMULATED: the p virtual
// ranks' buffers back to back on one GPU).
//
//   layouts (psize = n/p, the paper's names):
//     BLOCK    rank r holds x[r*psize + i]              (xblock)
//     CYCLIC   rank r holds x[r + p*j]                  (xcyclic)
//     CENTRAL  rank 0 holds all of x in natural order   (the paper's processor 0)
//   routes:
//     DIRECT   Fig 5.9 / Fig 5.3: every rank sends its slot
//              for every other rank -- m(m-1) messages of psize/m
//     CENTRAL  Fig 5.4: through processor 0 -- gather then scatter,
//              2(m-1) messages, every element moved twice, processor 0 the bottleneck
//
// Index algebra (q = psize/p):
//   BLOCK -> CYCLIC, direct:  rank r packs S_r[d][j] = b_r[d + p j]; S_r[d] -> rank d,
//                             slot r q (then out_d[r q + j] = x[d + p (r q + j)]).
//   CYCLIC -> BLOCK, direct:  c_d[a q + b] -> rank a, R_a[d][b]; unpack
//                             out_a[d + p b] = R_a[d q + b] (= x[a psize + d + p b]).
//   CENTRAL -> CYCLIC:        rank 0 packs S_0[r][j] = x[r + p j] (DISTRIBUTE_CENTRALIZED_
//                             TO_CYCLIC_PARTITIONED, Fig 5.8); S_0[r] -> rank r.
//   CYCLIC -> CENTRAL:        c_r -> rank 0, R_0[r]; unpack x[r + p j] = R_0[r n/p + j]
//                             (DISTRIBUTE_CYCLIC_PARTITIONED_TO_CENTRALIZED).
//   CENTRAL <-> BLOCK:        contiguous scatter / gather of the blocks.
//   via CENTRAL:              BLOCK -> CENTRAL (into rank 0's scratch) then CENTRAL -> CYCLIC,
//                             or CYCLIC -> CENTRAL (scratch) then CENTRAL -> BLOCK.
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "plan_internal.h"

namespace moa {

// The [q][P] <-> [P][q] transposes of the pack / unpack steps, tiled through shared
// memory so both global sides are contiguous: a CTA owns JT consecutive j, i.e. one
// contiguous run of JT*P interleaved elements and P runs of JT elements.  Shared slot
// of (j, d): j*P + (d ^ (j & (P-1))) -- the XOR spreads the P values of one d over the
// bank groups.
constexpr int XL_THREADS = 256;
constexpr int XL_ELEMS = 2048;   // elements per CTA tile (32 KiB)

// INTER = false: dst[d*q + j] = src[d + P*j] (deinterleave);  true: the inverse
template <int P, bool INTER>
__global__ void __launch_bounds__(XL_THREADS) xleave_kernel(const double2 *__restrict__ src,
                                                             double2 *__restrict__ dst, int64_t q) {
    constexpr int JT = XL_ELEMS / P;
    __shared__ double2 tile[XL_ELEMS];
    for (int64_t j0 = (int64_t)blockIdx.x * JT; j0 < q; j0 += (int64_t)gridDim.x * JT) {
        const int jn = (int)((q - j0) < JT ? (q - j0) : JT);
        if constexpr (!INTER) {
            const double2 *s = src + P * j0;   // contiguous run of jn*P elements
            for (int e = threadIdx.x; e < jn * P; e += XL_THREADS) {
                const int j = e / P, d = e % P;
                tile[j * P + (d ^ (j & (P - 1)))] = __ldg(s + e);
            }
            __syncthreads();
            for (int e = threadIdx.x; e < jn * P; e += XL_THREADS) {
                const int d = e / jn, j = e % jn;
                dst[d * q + j0 + j] = tile[j * P + (d ^ (j & (P - 1)))];
            }
        } else {
            for (int e = threadIdx.x; e < jn * P; e += XL_THREADS) {
                const int d = e / jn, j = e % jn;
                tile[j * P + (d ^ (j & (P - 1)))] = __ldg(src + d * q + j0 + j);
            }
            __syncthreads();
            double2 *o = dst + P * j0;
            for (int e = threadIdx.x; e < jn * P; e += XL_THREADS) {
                const int j = e / P, d = e % P;
                o[e] = tile[j * P + (d ^ (j & (P - 1)))];
            }
        }
        __syncthreads();
    }
}

static cudaError_t launch_xleave(bool inter, const double2 *src, double2 *dst, int p, int64_t q, cudaStream_t s) {
    if (q <= 0) return cudaSuccess;
    const int64_t jt = XL_ELEMS / p;
    int64_t blocks = (q + jt - 1) / jt;
    if (blocks > (int64_t)sm_count() * 6) blocks = (int64_t)sm_count() * 6;
#define MOA_XL(PP)                                                                                   \
    case PP:                                                                                         \
        if (inter) xleave_kernel<PP, true><<<(unsigned)blocks, XL_THREADS, 0, s>>>(src, dst, q);     \
        else xleave_kernel<PP, false><<<(unsigned)blocks, XL_THREADS, 0, s>>>(src, dst, q);          \
        break;
    switch (p) {
        MOA_XL(1)
        MOA_XL(2)
        MOA_XL(4)
        MOA_XL(8)
        MOA_XL(16)
    default: return cudaErrorInvalidValue;
    }
#undef MOA_XL
    return cudaGetLastError();
}

}  // namespace moa

using namespace moa;

// one transfer of a round: count elements from (rank src, buffer, offset) to (rank dst, ...)
enum RBuf { B_IN = 0, B_OUT = 1, B_S = 2, B_R = 3 };
struct Xfer {
    int src, dst;
    RBuf sb, db;
    int64_t so, doff, count;
};
// one step: a kernel on some ranks' buffers, or a round of transfers
struct Step {
    int kind;   // 0 = round, 1 = deinterleave, 2 = interleave
    std::vector<Xfer> xf;
    int rank;   // kernel steps: the rank whose buffers it touches (-1 = every rank)
    RBuf sb, db;
    int64_t q;  // kernel: q (P values per j)
};

struct moa_redist_s {
    int64_t n = 0, psize = 0;
    int p = 1, rank = 0, from = 0, to = 0, route = 0;
    bool emulated = false;
    int device = 0;
    cudaStream_t stream = nullptr;
    double2 *S = nullptr, *R = nullptr;   // scratch (per virtual rank: S_r at S + r*s_elems)
    int64_t s_elems = 0, r_elems = 0;
    int s_sets = 1, r_sets = 1;   // scratch sets allocated (p for per-rank scratch on virtual ranks)
    std::vector<Step> steps;
    int64_t messages = 0, bytes_max_rank = 0;
};

static int64_t elems_of(const moa_redist_s *pl, int layout, int r) {
    if (layout == MOA_LAYOUT_CENTRAL) return r == 0 ? pl->n : 0;
    return pl->psize;
}

static double2 *buf_of(moa_redist_s *pl, RBuf b, int r, const double2 *in, double2 *out) {
    const int vr = pl->emulated ? r : 0;   // real ranks own one set of buffers
    switch (b) {
    case B_IN: return const_cast<double2 *>(in) + (pl->emulated ? vr * (pl->from == MOA_LAYOUT_CENTRAL ? 0 : pl->psize) : 0);
    case B_OUT: return out + (pl->emulated ? vr * (pl->to == MOA_LAYOUT_CENTRAL ? 0 : pl->psize) : 0);
    case B_S: return pl->S + (pl->s_sets > 1 ? vr : 0) * pl->s_elems;
    default: return pl->R + (pl->r_sets > 1 ? vr : 0) * pl->r_elems;
    }
}

static int build_steps(moa_redist_s *pl) {
    const int p = pl->p;
    const int64_t n = pl->n, ps = pl->psize, q = ps / p, nq = n / p;
    auto round = [&]() -> Step & {
        pl->steps.push_back(Step{0, {}, -1, B_IN, B_OUT, 0});
        return pl->steps.back();
    };
    auto kern = [&](int kind, int rank, RBuf sb, RBuf db, int64_t qq) {
        pl->steps.push_back(Step{kind, {}, rank, sb, db, qq});
    };
    // building blocks (src buffer sb on the source side, db on the destination side)
    auto central_to_cyclic = [&](RBuf sb, RBuf db) {   // rank 0 packs into S_0, scatters
        kern(1, 0, sb, B_S, nq);
        Step &st = round();
        for (int r = 0; r < p; ++r) st.xf.push_back({0, r, B_S, db, r * nq, 0, nq});
    };
    auto cyclic_to_central = [&](RBuf sb, RBuf db) {   // gather into R_0, unpack on rank 0
        Step &st = round();
        for (int r = 0; r < p; ++r) st.xf.push_back({r, 0, sb, B_R, 0, r * nq, nq});
        kern(2, 0, B_R, db, nq);
    };
    auto block_to_central = [&](RBuf sb, RBuf db) {
        Step &st = round();
        for (int r = 0; r < p; ++r) st.xf.push_back({r, 0, sb, db, 0, r * ps, ps});
    };
    auto central_to_block = [&](RBuf sb, RBuf db) {
        Step &st = round();
        for (int r = 0; r < p; ++r) st.xf.push_back({0, r, sb, db, r * ps, 0, ps});
    };
    const int f = pl->from, t = pl->to;
    const bool via = pl->route == MOA_ROUTE_CENTRAL;
    pl->s_elems = pl->r_elems = 0;
    if (f == t) {
        Step &st = round();
        for (int r = 0; r < p; ++r)
            if (elems_of(pl, f, r)) st.xf.push_back({r, r, B_IN, B_OUT, 0, 0, elems_of(pl, f, r)});
    } else if (f == MOA_LAYOUT_BLOCK && t == MOA_LAYOUT_CYCLIC && !via) {
        pl->s_elems = ps;
        kern(1, -1, B_IN, B_S, q);
        Step &st = round();
        for (int r = 0; r < p; ++r)
            for (int d = 0; d < p; ++d) st.xf.push_back({r, d, B_S, B_OUT, d * q, r * q, q});
    } else if (f == MOA_LAYOUT_CYCLIC && t == MOA_LAYOUT_BLOCK && !via) {
        pl->r_elems = ps;
        Step &st = round();
        for (int d = 0; d < p; ++d)
            for (int a = 0; a < p; ++a) st.xf.push_back({d, a, B_IN, B_R, a * q, d * q, q});
        kern(2, -1, B_R, B_OUT, q);
    } else if (f == MOA_LAYOUT_CENTRAL && t == MOA_LAYOUT_CYCLIC) {
        pl->s_elems = n;
        central_to_cyclic(B_IN, B_OUT);
    } else if (f == MOA_LAYOUT_CYCLIC && t == MOA_LAYOUT_CENTRAL) {
        pl->r_elems = n;
        cyclic_to_central(B_IN, B_OUT);
    } else if (f == MOA_LAYOUT_CENTRAL && t == MOA_LAYOUT_BLOCK) {
        central_to_block(B_IN, B_OUT);
    } else if (f == MOA_LAYOUT_BLOCK && t == MOA_LAYOUT_CENTRAL) {
        block_to_central(B_IN, B_OUT);
    } else if (f == MOA_LAYOUT_BLOCK && t == MOA_LAYOUT_CYCLIC && via) {
        // Fig 5.4: the blocks gathered on processor 0 (R_0 = x), then scattered cyclically
        pl->s_elems = pl->r_elems = n;
        block_to_central(B_IN, B_R);
        central_to_cyclic(B_R, B_OUT);
    } else if (f == MOA_LAYOUT_CYCLIC && t == MOA_LAYOUT_BLOCK && via) {
        pl->s_elems = pl->r_elems = n;
        cyclic_to_central(B_IN, B_S);   // x in natural order in S_0
        central_to_block(B_S, B_OUT);
    } else {
        return fail(MOA_ERR_INVALID_ARG, "unsupported redistribution %d -> %d (route %d)", f, t, pl->route);
    }
    // message and byte counts (messages = transfers between distinct ranks)
    std::vector<int64_t> sent(p, 0);
    for (const Step &st : pl->steps)
        for (const Xfer &x : st.xf)
            if (x.src != x.dst) {
                pl->messages += 1;
                sent[x.src] += 16 * x.count;
            }
    for (int r = 0; r < p; ++r) pl->bytes_max_rank = sent[r] > pl->bytes_max_rank ? sent[r] : pl->bytes_max_rank;
    return MOA_OK;
}

static int run_steps(moa_redist_s *pl, const double2 *in, double2 *out) {
    const int p = pl->p;
    cudaStream_t s = pl->stream;
    for (const Step &st : pl->steps) {
        if (st.kind != 0) {
            for (int r = 0; r < p; ++r) {
                if (st.rank >= 0 && st.rank != r) continue;
                if (!pl->emulated && r != pl->rank) continue;
                CUDA_TRY(launch_xleave(st.kind == 2, buf_of(pl, st.sb, r, in, out), buf_of(pl, st.db, r, in, out), p,
                                       st.q, s));
            }
            continue;
        }
        if (pl->emulated) {   // every transfer is a device copy
            for (const Xfer &x : st.xf)
                CUDA_TRY(cudaMemcpyAsync(buf_of(pl, x.db, x.dst, in, out) + x.doff, buf_of(pl, x.sb, x.src, in, out) + x.so,
                                         x.count * sizeof(double2), cudaMemcpyDeviceToDevice, s));
            continue;
        }
        std::vector<const double2 *> sp(p, nullptr);
        std::vector<double2 *> rp(p, nullptr);
        std::vector<int64_t> sn(p, 0), rn(p, 0);
        for (const Xfer &x : st.xf) {
            if (x.src == pl->rank) {
                sp[x.dst] = buf_of(pl, x.sb, x.src, in, out) + x.so;
                sn[x.dst] = x.count;
            }
            if (x.dst == pl->rank) {
                rp[x.src] = buf_of(pl, x.db, x.dst, in, out) + x.doff;
                rn[x.src] = x.count;
            }
        }
        std::string err;
        int rc = dist_sendrecv(sp.data(), sn.data(), rp.data(), rn.data(), p, pl->rank, s, &err);
        if (rc) return fail(rc, "%s", err.c_str());
    }
    return MOA_OK;
}

extern "C" {

moa_redist_t moa_redist_plan(int64_t n, int p, int from, int to, int route, int mode) {
    clear_error();
    if (!pow2(n) || n < 2 || n > ((int64_t)1 << 32)) {
        fail(MOA_ERR_INVALID_N, "n=%lld must be 2^t with 1 <= t <= 32 (Fig 2.1: n = 2^t, t >= 1)", (long long)n);
        return nullptr;
    }
    if (!pow2(p) || p > 16 || n / p < p) {
        fail(MOA_ERR_INVALID_P, "p=%d must be a power of two <= 16 with psize = n/p >= p (P:289)", p);
        return nullptr;
    }
    if (from < MOA_LAYOUT_BLOCK || from > MOA_LAYOUT_CENTRAL || to < MOA_LAYOUT_BLOCK || to > MOA_LAYOUT_CENTRAL ||
        (route != MOA_ROUTE_DIRECT && route != MOA_ROUTE_CENTRAL) ||
        (mode != MOA_MODE_LIFTED && mode != MOA_MODE_EMULATED)) {
        fail(MOA_ERR_INVALID_ARG, "bad layout (%d -> %d), route %d or mode %d", from, to, route, mode);
        return nullptr;
    }
    moa_redist_s *pl = new moa_redist_s();
    pl->n = n;
    pl->p = p;
    pl->psize = n / p;
    pl->from = from;
    pl->to = to;
    pl->route = route;
    pl->emulated = mode == MOA_MODE_EMULATED || p == 1;   // p = 1: every transfer is a local copy
    cudaGetDevice(&pl->device);
    if (!pl->emulated && p > 1) {
        int wr = -1, ws = 0;
        if (dist_world(&wr, &ws) != MOA_OK || ws == 0) {
            delete pl;
            fail(MOA_ERR_NO_DIST, "p=%d > 1 needs moa_dist_init first (or MOA_MODE_EMULATED)", p);
            return nullptr;
        }
        if (ws != p) {
            delete pl;
            fail(MOA_ERR_INVALID_P, "p=%d differs from the world size %d", p, ws);
            return nullptr;
        }
        pl->rank = wr;
    }
    if (build_steps(pl) != MOA_OK) {
        delete pl;
        return nullptr;
    }
    // scratch: psize-element S/R on every rank for the direct block <-> cyclic routes (p sets
    // on virtual ranks); the n-element ones of the central routes only on processor 0
    const bool s_central = pl->s_elems == n, r_central = pl->r_elems == n;
    const int s_sets = pl->emulated && !s_central ? p : 1, r_sets = pl->emulated && !r_central ? p : 1;
    pl->s_sets = s_sets;
    pl->r_sets = r_sets;
    const bool need_s = pl->s_elems > 0 && (pl->emulated || !s_central || pl->rank == 0);
    const bool need_r = pl->r_elems > 0 && (pl->emulated || !r_central || pl->rank == 0);
    if ((need_s && cudaMalloc((void **)&pl->S, (size_t)pl->s_elems * s_sets * sizeof(double2)) != cudaSuccess) ||
        (need_r && cudaMalloc((void **)&pl->R, (size_t)pl->r_elems * r_sets * sizeof(double2)) != cudaSuccess)) {
        cudaGetLastError();
        cudaFree(pl->S);
        delete pl;
        fail(MOA_ERR_OOM, "redistribution scratch allocation failed");
        return nullptr;
    }
    return pl;
}

int moa_redist_execute(moa_redist_t pl, const void *in, void *out) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL redistribution plan");
    const bool in_needed = pl->emulated ? true : elems_of(pl, pl->from, pl->rank) > 0;
    const bool out_needed = pl->emulated ? true : elems_of(pl, pl->to, pl->rank) > 0;
    if ((in_needed && !aligned16(in)) || (out_needed && !aligned16(out)))
        return fail(MOA_ERR_ALIGN, "in/out must be 16-byte aligned device pointers (NULL only where the layout "
                                   "gives this rank no elements)");
    if (in_needed && out_needed && in == out)
        return fail(MOA_ERR_INVALID_ARG, "redistribution is out of place (in != out)");
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != pl->device) cudaSetDevice(pl->device);
    int rc = run_steps(pl, (const double2 *)in, (double2 *)out);
    if (cur != pl->device) cudaSetDevice(cur);
    return rc;
}

int moa_redist_set_stream(moa_redist_t pl, void *stream) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL redistribution plan");
    pl->stream = (cudaStream_t)stream;
    return MOA_OK;
}

int moa_redist_info(moa_redist_t pl, int64_t *messages, int64_t *max_rank_bytes, int64_t *elems_in,
                    int64_t *elems_out) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL redistribution plan");
    if (messages) *messages = pl->messages;
    if (max_rank_bytes) *max_rank_bytes = pl->bytes_max_rank;
    const int r = pl->rank;
    if (elems_in) *elems_in = pl->emulated ? pl->n : elems_of(pl, pl->from, r);
    if (elems_out) *elems_out = pl->emulated ? pl->n : elems_of(pl, pl->to, r);
    return MOA_OK;
}

void moa_redist_destroy(moa_redist_t pl) {
    if (!pl) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(pl->device);
    cudaStreamSynchronize(pl->stream);
    cudaFree(pl->S);
    cudaFree(pl->R);
    cudaSetDevice(cur);
    delete pl;
}

}  // extern "C"
