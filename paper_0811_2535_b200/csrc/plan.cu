// plan.cu -- plan builder (dimension lifting + FP64 twiddle tables), executor
// and the C ABI declared in include/moa_fft.h.
//
// Plan = the paper's Phase 3/4 artefacts made concrete for B200:
//   S0 validation and lifting   n = 2^t, psize = n/p >= p, breakpoint =
//                               log2(psize)+1 (the high end of §4.8)
//   S1 twiddle tables           built once per plan in long double (the paper
//                               recomputes weight(row) every stage)
//   S3/S4 lifted passes         one PassDesc per level of <F1..Fd>
//   S5/S6 (p > 1)               the local psize-point FFT whose last pass scales by
//                               omega_n^(r*k1) and packs for the all-to-all (Fig 5.9)
//   S7 all-to-all               NCCL grouped send/recv (dist.cu)
//   S8 cyclic phase             pcombine<P>
#include <dlfcn.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/moa_fft.h"
#include "moa_internal.h"

namespace moa {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return fail(MOA_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                               \
    } while (0)

// ------------------------------------------------------------------ NCCL (dist.cu)
int dist_world(int *rank, int *size);
int dist_alltoall(const double2 *send, double2 *recv, int64_t chunk, int p, int rank, cudaStream_t s,
                  std::string *err);
int dist_barrier(cudaStream_t s, std::string *err);
int dist_allgather_sync(const void *send_dev, void *recv_dev, size_t bytes, cudaStream_t s, std::string *err);

// ------------------------------------------------------------------ twiddles
// exp(-2 pi i e / N) for N a power of two, evaluated in long double on the
// first octant of the circle and rounded once to double; quarter turns exact.
static double2 host_root(uint64_t e, uint64_t N) {
    e &= N - 1;
    // position on the circle in units of N/8 (octant) with remainder
    unsigned __int128 e8 = (unsigned __int128)e * 8;
    int oct = (int)(e8 / N);
    uint64_t rem = (uint64_t)(e8 % N);  // angle inside the octant = (pi/4) * rem / N
    const long double quarter_pi = 0.785398163397448309615660845819875721L;
    long double a = quarter_pi * ((long double)rem / (long double)N);
    long double b = quarter_pi - a;  // complementary angle within the octant
    long double c, s;
    // cos/sin of theta = oct*pi/4 + a using only angles in [0, pi/4]
    switch (oct) {
    case 0: c = cosl(a); s = sinl(a); break;
    case 1: c = sinl(b); s = cosl(b); break;
    case 2: c = -sinl(a); s = cosl(a); break;
    case 3: c = -cosl(b); s = sinl(b); break;
    case 4: c = -cosl(a); s = -sinl(a); break;
    case 5: c = -sinl(b); s = -cosl(b); break;
    case 6: c = sinl(a); s = -cosl(a); break;
    default: c = cosl(b); s = -sinl(b); break;
    }
    return make_double2((double)c, (double)(-s));
}

// ------------------------------------------------------------------ plan
struct PassPlan {
    int logF, T;
    int64_t tiles;
    PassDesc d;  // src/dst patched at execute
    // TMA-staged persistent variant (0 = plain kernel, 1 = column tile, 2 = row tile)
    int tma = 0;
    int tma_grid = 0;
    int pf_grid = 0;   // > 0: prefetching persistent kernel (fft_pass_pf_kernel)
    int io = 0;        // r-D axis passes: 0 = out -> out (in place), 1 = out -> work, 2 = work -> out
    CUtensorMap map;
    const void *map_base = nullptr;
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// The box geometry must match TmaShape / tma_issue_tile in fft_pass.cuh.
static int encode_pass_map(PassPlan &pp, const void *base) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return fail(MOA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const PassDesc &D = pp.d;
    const uint64_t F = 1ull << pp.logF, T = pp.T;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
    cuuint32_t rank;
    if (pp.tma == 1 || pp.tma == 4) {   // column tile of the view [A][F][B]: dims {2B doubles, F, A}
        const uint64_t B = (uint64_t)D.in_f, A = (uint64_t)D.V;
        rank = 3;
        dims[0] = 2 * B;
        dims[1] = F;
        dims[2] = A;
        strides[0] = 16 * B;
        strides[1] = 16 * F * B;
        box[0] = (cuuint32_t)(2 * T);
        box[1] = (cuuint32_t)(F < 256 ? F : 256);
        box[2] = 1;
    } else {             // row tile: dims {2F doubles, rows (u*T + t), V, W}
        const uint64_t rows = (uint64_t)D.U * T, V = (uint64_t)D.V, W = (uint64_t)(pp.tiles / (D.U * D.V));
        rank = 4;
        dims[0] = 2 * F;
        dims[1] = rows;
        dims[2] = V;
        dims[3] = W;
        strides[0] = 16 * (uint64_t)D.in_t;
        strides[1] = 16 * (uint64_t)(D.in_v ? D.in_v : D.in_t * rows);
        strides[2] = 16 * (uint64_t)(D.in_w ? D.in_w : D.in_t * rows * V);
        box[0] = (cuuint32_t)(F < 128 ? 2 * F : 256);
        box[1] = (cuuint32_t)T;
        box[2] = 1;
        box[3] = 1;
    }
    CUresult r = enc(&pp.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void *>(base), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(MOA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for pass F=%llu T=%llu", (int)r,
                                       (unsigned long long)F, (unsigned long long)T);
    pp.map_base = base;
    return MOA_OK;
}

// choose the TMA-staged variant when it exists for this (F, T, layout), else the
// prefetching persistent kernel when selected
static void choose_tma(PassPlan &pp) {
    pp.tma = 0;
    pp.pf_grid = 0;
    const char *pf_env = getenv("MOA_FFT_PF");
    if (pf_env && atoi(pf_env) && pp.logF >= 5) {
        int g = pass_pf_grid(pp.logF, pp.T);
        if (g > 0) pp.pf_grid = (int)(g < pp.tiles ? g : pp.tiles);
    }
    const char *tma_env = getenv("MOA_FFT_TMA");   // 1: double-buffered TMA, 2: single buffer + prefetch
    if (!tma_env || atoi(tma_env) == 0) return;
    const int tma_kind = atoi(tma_env);
    const PassDesc &D = pp.d;
    int src = 0;
    if (!D.last && D.in_t == 1 && pp.T >= 2) src = 1;
    else if (D.last && D.in_f == 1) src = 2;
    if (!src) return;
    const int code = tma_kind == 2 ? src + 3 : src;
    int g = pass_tma_grid(pp.logF, pp.T, code);
    if (g <= 0) return;
    pp.tma = code;
    pp.tma_grid = g;
}

}  // namespace moa

using namespace moa;

struct moa_fft_plan_s {
    int64_t n = 0, M = 0;
    int64_t batch = 1;   // independent transforms per execute (p == 1)
    // 2-D plans (moa_fft_plan_2d): rows = batched 1-D plan of length n2, col = one pass
    // of n1-point DFTs along the stride-n2 axis, in place on the output
    int64_t n1 = 0, n2 = 0;
    moa_fft_plan_s *rows = nullptr;
    int t = 0, p = 1, rank = 0, sign = -1, mode = MOA_MODE_LIFTED;
    int d = 0;
    int64_t lift[4] = {0, 0, 0, 0};
    int chunks = 1;
    int exchange = MOA_XCHG_NCCL;
    // P2P exchange: receive buffers of every rank (own = recv), double-buffered per execute
    double2 *peer_recv[16] = {};
    bool peer_mapped[16] = {};   // opened through cudaIpcOpenMemHandle (closed in destroy)
    bool peers_open = false;
    int next_phase = 1;
    unsigned long long xbuf = 0;   // which half of the receive buffers this execute uses
    int device = 0;
    int hbits = 0;
    cudaStream_t stream = nullptr;
    double2 *tw_hi = nullptr, *tw_lo = nullptr, *tw_f = nullptr;
    std::vector<double2 *> axis_tw;   // r-D plans: two-level omega_N tables of lifted non-last axes
    double2 *work = nullptr, *send = nullptr, *recv = nullptr;
    double2 *stage_in = nullptr, *stage_out = nullptr;  // execute_host staging
    // execute_host_batch: second staging pair + copy streams and events (lazily created)
    double2 *stage_in2 = nullptr, *stage_out2 = nullptr;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
    int64_t work_elems = 0, send_elems = 0;
    std::vector<PassPlan> passes;   // p == 1: all passes; p > 1: phase 1 for rank `rank`; 2-D: the column pass
    std::vector<std::vector<PassPlan>> rank_passes;  // emulated: phase 1 per virtual rank
    int64_t workspace_bytes = 0;
    // L2-fused last two passes (fused.cu)
    bool fused = false;
    FusedDesc fd;
    CUtensorMap fmap2, fmap3;
    int fgrid = 0;
    int *items = nullptr;
    unsigned long long *counters = nullptr;
    double2 *scratch = nullptr;
    unsigned long long epoch = 0;
    // per-kernel event profiling (moa_fft_set_profiling)
    bool profiling = false;
    struct Slot {
        std::string name;
        int64_t bytes;
        int launches;
        double ms;
    };
    struct Rec {
        int slot;
        cudaEvent_t a, b;
    };
    std::vector<Slot> slots;
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
};

namespace moa {

static int ilog2(int64_t v) {
    int r = 0;
    while (((int64_t)1 << r) < v) ++r;
    return r;
}
static bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

static int env_int(const char *name, int dflt) {
    const char *s = getenv(name);
    return (s && *s) ? atoi(s) : dflt;
}

// default lifting <F1..Fd> of a local length 2^tl, from the B200 lifting sweeps
// (tools/perf_probe.py): 256-point passes (4 tiles per SM) wherever the
// length allows, the remaining factor in the row pass up to 2^12, four levels from 2^29
// on (two <= 128-point column passes instead of one long one).  p > 1 plans keep <= 3
// levels.
static int default_lifting(int tl, int64_t *lift, int p) {
    if (tl <= FMAX_LOG) {
        lift[0] = (int64_t)1 << tl;
        return 1;
    }
    if (tl <= 20) {   // two levels, the longer one last: <256,256> at 2^16, <1024,1024> at 2^20
        int a = tl / 2;
        lift[0] = (int64_t)1 << a;
        lift[1] = (int64_t)1 << (tl - a);
        return 2;
    }
    if (tl >= 25 && tl <= 28) {   // <256, 256, 2^(tl-16)>: the long factor in the row pass
        lift[0] = 256;
        lift[1] = 256;
        lift[2] = (int64_t)1 << (tl - 16);
        return 3;
    }
    if (tl <= 27 || (p > 1 && tl <= 16 + FMAX_LOG)) {   // <2^(tl-16), 256, 256>
        lift[0] = (int64_t)1 << (tl - 16);
        lift[1] = 256;
        lift[2] = 256;
        return 3;
    }
    if (tl <= 16 + 2 * 8 && p == 1) {   // <a, b, 256, 256>, a <= b <= 256
        int a = (tl - 16) / 2;
        lift[0] = (int64_t)1 << a;
        lift[1] = (int64_t)1 << (tl - 16 - a);
        lift[2] = 256;
        lift[3] = 256;
        return 4;
    }
    if (tl <= 3 * FMAX_LOG) {
        int a = tl / 3, b = (tl - a) / 2;
        lift[0] = (int64_t)1 << a;
        lift[1] = (int64_t)1 << b;
        lift[2] = (int64_t)1 << (tl - a - b);
        return 3;
    }
    int a = tl / 4, b = (tl - a) / 3, c = (tl - a - b) / 2;
    lift[0] = (int64_t)1 << a;
    lift[1] = (int64_t)1 << b;
    lift[2] = (int64_t)1 << c;
    lift[3] = (int64_t)1 << (tl - a - b - c);
    return 4;
}

static int choose_T(int logF, int64_t avail) {
    // tile size cap: long transforms take T*F = 8192 (one 128 KiB tile per SM);
    // short ones 4096 (2-3 tiles per SM overlap memory and FP64 work)
    // measured on B200 (tools/perf_probe.py): 2048-element tiles (4 CTAs/SM) for F <= 256,
    // 4096 for F = 512 .. 2048 (T = 8, 4, 2), one 8192 tile above
    int tf_max = env_int("MOA_FFT_TF", logF >= 12 ? TF_MAX : (logF >= 9 ? 4096 : 2048));
    if (tf_max > TF_MAX) tf_max = TF_MAX;
    int T = 1;
    while (T < 64 && ((int64_t)(2 * T) << logF) <= tf_max && 2 * T <= avail) T *= 2;
    while (T > 1 && !pass_supported(logF, T)) T /= 2;
    return T;
}

// Build the passes of a local FFT of length M = prod(lift) (global length n).
// rank >= 0 with P > 1: the last pass scales by omega_n^(rank*K) and packs to
// the send layout [dst][c] with K = dst + P*c (S6, fused into S4's epilogue).
static int build_passes(const moa_fft_plan_s *pl, int rank, int P, std::vector<PassPlan> &out) {
    const int d = pl->d;
    const int64_t *Fv = pl->lift;
    const int64_t n = pl->n;
    out.clear();
    for (int i = 0; i < d; ++i) {
        PassPlan pp;
        memset(&pp.d, 0, sizeof(PassDesc));
        PassDesc &D = pp.d;
        const int64_t F = Fv[i];
        int64_t A = 1, B = 1;
        for (int l = 0; l < i; ++l) A *= Fv[l];
        for (int l = i + 1; l < d; ++l) B *= Fv[l];
        pp.logF = ilog2(F);
        D.nmask = (uint64_t)n - 1;
        D.hbits = pl->hbits;
        D.tbits = pl->t;
        D.tw_hi = pl->tw_hi;
        D.tw_lo = pl->tw_lo;
        D.tw_f = pl->tw_f;
        D.pack_lp = -1;
        D.conj_in = (i == 0 && pl->sign > 0);
        D.conj_out = 0;
        if (i < d - 1) {
            // middle pass: view [A][F][B], F-point DFTs along the middle axis for
            // every (a, b); twiddle omega_{F*B}^(b*k) = omega_n^(b*k*n/(F*B)); in place.
            int T = choose_T(pp.logF, B);
            pp.T = T;
            D.U = B / T;
            D.V = A;
            D.in_u = T;
            D.in_v = F * B;
            D.in_t = 1;
            D.in_f = B;
            int64_t mult = n / (F * B);
            D.twiddle = 1;
            D.b_u = mult * T;
            D.b_t = mult;
            D.in_tfast = T > 1;
            D.out_tfast = T > 1;
            D.last = 0;
            D.out_u = D.in_u;
            D.out_v = D.in_v;
            D.out_w = D.in_w;
            D.out_t = D.in_t;
            D.out_k = D.in_f;
            pp.tiles = D.U * D.V;
        } else {
            // last pass: rows of length F indexed by the digits (k_0 .. k_{d-2}) the
            // earlier passes produced (k_0 most significant); output index
            // K = k_0 + F_0 k_1 + F_0 F_1 k_2 + ... + (F_0..F_{d-2}) k : the
            // transpose <d-1 .. 0> + ravel of Fig A.1, i.e. natural order.
            D.last = 1;
            D.in_f = 1;
            D.in_tfast = 0;
            int64_t S[3] = {0, 0, 0};   // stride (in rows) of digit k_l in the row index
            for (int l = 0; l < d - 1; ++l) {
                int64_t s = 1;
                for (int m = l + 1; m < d - 1; ++m) s *= Fv[m];
                S[l] = s;
            }
            int64_t Kk = A;
            int64_t K_d1 = d >= 3 ? Fv[0] : 0;      // weight of k_1
            int64_t K_d2 = d >= 4 ? Fv[0] * Fv[1] : 0;
            if (d == 1) {
                pp.T = 1;
                D.U = 1;
                D.V = 1;
                D.K_k = 1;
                D.out_tfast = 0;
                pp.tiles = 1;
                if (P > 1) {
                    D.pack_lp = ilog2(P);
                    D.pack_chunk = pl->M / P;
                }
            } else if (P > 1) {
                if (d > 3) return fail(MOA_ERR_INVALID_ARG, "p > 1 supports lifting depth <= 3");
                // rows k_0 = dst + P*(cb*T + t): every row of a tile goes to one destination
                int T = choose_T(pp.logF, Fv[0] / P);
                pp.T = T;
                D.U = Fv[0] / (P * T);
                D.V = P;
                D.in_u = P * T * S[0] * F;
                D.in_v = S[0] * F;
                D.in_t = P * S[0] * F;
                D.in_w = d >= 3 ? S[1] * F : 0;
                D.K_u = P * T;
                D.K_v = 1;
                D.K_t = P;
                D.K_w = K_d1;
                D.K_k = Kk;
                D.out_tfast = T > 1;
                D.pack_lp = ilog2(P);
                D.pack_chunk = pl->M / P;
                pp.tiles = D.U * D.V * (d >= 3 ? Fv[1] : 1);
            } else {
                int T = choose_T(pp.logF, Fv[0]);
                pp.T = T;
                D.U = Fv[0] / T;
                D.V = d >= 3 ? Fv[1] : 1;
                D.in_u = T * S[0] * F;
                D.in_t = S[0] * F;
                D.in_v = d >= 3 ? S[1] * F : 0;
                D.in_w = d >= 4 ? S[2] * F : 0;
                D.K_u = T;
                D.K_t = 1;
                D.K_v = K_d1;
                D.K_w = K_d2;
                D.K_k = Kk;
                D.out_tfast = T > 1;
                pp.tiles = D.U * D.V * (d >= 4 ? Fv[2] : 1);
            }
            if (P > 1 && rank > 0) {
                // S6: Y_r[K] <- omega_n^(r*K) Y_r[K]  (weightcyclic, Fig 4.4)
                uint64_t r = (uint64_t)rank;
                D.twiddle = 1;
                D.a_u = (int64_t)(r * (uint64_t)D.K_u);
                D.a_v = (int64_t)(r * (uint64_t)D.K_v);
                D.a_w = (int64_t)(r * (uint64_t)D.K_w);
                D.a_t = (int64_t)(r * (uint64_t)D.K_t);
                D.b_c = (int64_t)(r * (uint64_t)D.K_k);
            }
            D.conj_out = (P == 1 && pl->sign > 0);
            if (P == 1) {
                D.out_u = D.K_u;
                D.out_v = D.K_v;
                D.out_w = D.K_w;
                D.out_t = D.K_t;
                D.out_k = D.K_k;
            } else if (d > 1) {
                // send slot of K = dst + P*c is dst*chunk + K/P; with the tile rows
                // k_0 = dst + P*(u*T + t) every coefficient but v's is a multiple of P
                D.pack_lp = -1;
                D.out_u = D.K_u / P;
                D.out_v = pl->M / P;
                D.out_w = D.K_w / P;
                D.out_t = D.K_t / P;
                D.out_k = D.K_k / P;
            }
        }
        if (pl->batch > 1) {
            if (d == 1) {
                // tiles of T whole transforms (rows of n elements), one tile per group of T;
                // measured (tools/batch_probe.py): one transform per CTA from F = 1024 on
                int T = pp.logF >= 10 ? 1 : choose_T(pp.logF, pl->batch & -pl->batch);
                pp.T = T;
                D.in_t = pl->n;
                D.out_t = pl->n;
                D.out_tfast = 0;
                D.ltiles = 0;
                D.bstride = (int64_t)T * pl->n;
                pp.tiles = pl->batch / T;
            } else {
                int lt = ilog2(pp.tiles);
                D.ltiles = lt;
                D.bstride = pl->n;
                pp.tiles *= pl->batch;
            }
        }
        D.pdl = env_int("MOA_FFT_PDL", 1);   // measured: 2^24 275.5 -> 271.4 us, 2^16 15.3 -> 13.3 us
        if (!pow2(D.U) || !pow2(D.V))
            return fail(MOA_ERR_INVALID_ARG, "internal: tile grid %lld x %lld not powers of two", (long long)D.U,
                        (long long)D.V);
        D.lU = ilog2(D.U);
        D.lV = ilog2(D.V);
        if (!pass_supported(pp.logF, pp.T))
            return fail(MOA_ERR_INVALID_ARG, "no pass kernel for F=2^%d T=%d", pp.logF, pp.T);
        out.push_back(pp);
    }
    return MOA_OK;
}

static void free_plan(moa_fft_plan_s *pl) {
    if (!pl) return;
    if (pl->rows) {
        free_plan(pl->rows);
        pl->rows = nullptr;
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(pl->device);
    cudaStreamSynchronize(pl->stream);
    for (int r = 0; r < 16; ++r)
        if (pl->peer_mapped[r]) cudaIpcCloseMemHandle(pl->peer_recv[r]);
    for (double2 *p : pl->axis_tw) cudaFree(p);
    cudaFree(pl->tw_hi);
    cudaFree(pl->tw_lo);
    cudaFree(pl->tw_f);
    cudaFree(pl->work);
    cudaFree(pl->send);
    cudaFree(pl->recv);
    cudaFree(pl->stage_in);
    cudaFree(pl->stage_out);
    cudaFree(pl->stage_in2);
    cudaFree(pl->stage_out2);
    if (pl->h2d) cudaStreamSynchronize(pl->h2d), cudaStreamDestroy(pl->h2d);
    if (pl->d2h) cudaStreamSynchronize(pl->d2h), cudaStreamDestroy(pl->d2h);
    for (int b = 0; b < 2; ++b)
        for (cudaEvent_t e : {pl->ev_h2d[b], pl->ev_comp[b], pl->ev_d2h[b]})
            if (e) cudaEventDestroy(e);
    cudaFree(pl->items);
    cudaFree(pl->counters);
    cudaFree(pl->scratch);
    for (auto &r : pl->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : pl->pool) cudaEventDestroy(e);
    cudaSetDevice(cur);
    delete pl;
}

// Fuse the last two passes of a 3-level lifting through an L2-resident ring
// (fused.cu) when a kernel for their (F, T) pair exists; otherwise keep them separate.
static int setup_fused(moa_fft_plan_s *pl, int kind) {
    PassPlan &p2 = pl->passes[1], &p3 = pl->passes[2];
    if (!fused_supported(p2.logF, p2.T, p3.logF, p3.T)) return MOA_OK;
    const int64_t F1 = pl->lift[0], F2 = pl->lift[1], F3 = pl->lift[2];
    const int T3 = p3.T;
    const int groups = (int)(F1 / T3);
    const int tiles2 = (int)(F3 / p2.T) * T3;
    const int tiles3 = (int)F2;
    if (groups >= (1 << 14) || tiles2 >= (1 << 16) || tiles3 >= (1 << 16)) return MOA_OK;
    const bool ticket = kind >= 2;   // 2: blockIdx tickets, 3: atomic tickets
    int slots = env_int("MOA_FFT_SLOTS", ticket ? 4 : 3), lag = env_int("MOA_FFT_LAG", ticket ? 2 : 1);
    if (lag < 0) lag = 0;
    if (slots < lag + 1) slots = lag + 1;
    if (slots > groups) slots = groups;
    if (lag > slots - 1) lag = slots - 1;
    std::vector<int> items;
    for (int i = 0; i < groups + lag; ++i) {
        if (i < groups)
            for (int l = 0; l < tiles2; ++l) items.push_back((0 << 30) | (i << 16) | l);
        if (i - lag >= 0)
            for (int l = 0; l < tiles3; ++l) items.push_back((1 << 30) | ((i - lag) << 16) | l);
    }
    const int64_t group_elems = (int64_t)T3 * F2 * F3;
    if (cudaMalloc((void **)&pl->items, items.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc((void **)&pl->counters, (1 + 2 * (size_t)groups) * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc((void **)&pl->scratch, (size_t)slots * group_elems * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        return fail(MOA_ERR_OOM, "fused-pass buffers allocation failed");
    }
    pl->workspace_bytes += items.size() * sizeof(int) + (1 + 2 * groups) * 8 + slots * group_elems * 16;
    CUDA_TRY(cudaMemcpy(pl->items, items.data(), items.size() * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemset(pl->counters, 0, (1 + 2 * (size_t)groups) * sizeof(unsigned long long)));
    FusedDesc &fd = pl->fd;
    memset(&fd, 0, sizeof fd);
    fd.p2 = p2.d;
    fd.p3 = p3.d;
    fd.items = pl->items;
    fd.total_items = (int64_t)items.size();
    fd.claim = pl->counters;
    fd.done2 = pl->counters + 1;
    fd.done3 = pl->counters + 1 + groups;
    fd.tiles2 = tiles2;
    fd.tiles3 = tiles3;
    fd.groups = groups;
    fd.slots = slots;
    fd.rows_per_group_elems = group_elems;
    fd.scratch = pl->scratch;
    fd.f2f3 = F2 * F3;
    fd.discard = env_int("MOA_FFT_DISCARD", 1);
    fd.ticket = ticket ? kind - 1 : 0;
    {   // TMA maps: middle-pass column tiles over `work`, last-pass row tiles over the ring
        PassPlan tmp = p2;
        tmp.tma = 1;
        int rc = encode_pass_map(tmp, pl->work);
        if (rc) return rc;
        pl->fmap2 = tmp.map;
        EncodeTiledFn enc = encode_fn();
        cuuint64_t dims[4] = {(cuuint64_t)(2 * F3), (cuuint64_t)T3, (cuuint64_t)F2, (cuuint64_t)slots};
        cuuint64_t strides[3] = {(cuuint64_t)(16 * F2 * F3), (cuuint64_t)(16 * F3), (cuuint64_t)(16 * group_elems)};
        cuuint32_t box[4] = {(cuuint32_t)(F3 < 128 ? 2 * F3 : 256), (cuuint32_t)T3, 1, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = enc(&pl->fmap3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, pl->scratch, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(MOA_ERR_CUDA, "scratch tensor map encode failed (%d)", (int)r);
    }
    pl->fgrid = ticket ? (int)items.size() : fused_grid(p2.logF, p2.T, p3.logF, p3.T);
    int gmax = env_int("MOA_FFT_FGRID", 0);
    if (gmax > 0 && gmax < pl->fgrid) pl->fgrid = gmax;
    if (pl->fgrid <= 0) return fail(MOA_ERR_CUDA, "fused kernel occupancy query failed");
    pl->fused = true;
    return MOA_OK;
}

// lifting <F1..Fd> from the options or the default table; sets pl->lift, pl->d
static int resolve_lifting(moa_fft_plan_s *pl, const moa_fft_options *opt) {
    int tl = ilog2(pl->M);
    const int p = pl->p;
    if (opt && opt->nlift > 0) {
        if (opt->nlift > 4) return fail(MOA_ERR_INVALID_ARG, "lifting depth %d > 4", opt->nlift);
        int64_t prod = 1;
        for (int i = 0; i < opt->nlift; ++i) {
            int64_t F = opt->lift[i];
            if (!pow2(F) || F < 2 || F > FMAX)
                return fail(MOA_ERR_INVALID_ARG, "lifting factor %lld outside powers of two in [2, %d]",
                            (long long)F, FMAX);
            pl->lift[i] = F;
            prod *= F;
        }
        if (prod != pl->M)
            return fail(MOA_ERR_INVALID_ARG, "lifting product %lld != local length %lld", (long long)prod,
                        (long long)pl->M);
        pl->d = opt->nlift;
    } else {
        pl->d = default_lifting(tl, pl->lift, p);
    }
    if (p > 1 && pl->lift[0] < p && pl->d > 1)
        return fail(MOA_ERR_INVALID_ARG, "first lifting factor %lld < p=%d", (long long)pl->lift[0], p);
    return MOA_OK;
}

static int make_plan(int64_t n, int p, int sign, const moa_fft_options *opt, moa_fft_plan_s **res) {
    *res = nullptr;
    int mode = opt ? opt->mode : MOA_MODE_LIFTED;
    if (!pow2(n) || n < 2 || n > ((int64_t)1 << 32))
        return fail(MOA_ERR_INVALID_N, "n=%lld must be 2^t with 1 <= t <= 32 (Fig 2.1: n = 2^t, t >= 1)",
                    (long long)n);
    if (sign != -1 && sign != 1) return fail(MOA_ERR_INVALID_SIGN, "sign=%d must be -1 or +1", sign);
    if (mode < MOA_MODE_LIFTED || mode > MOA_MODE_EMULATED)
        return fail(MOA_ERR_INVALID_ARG, "unknown mode %d", mode);
    if (!pow2(p) || p > 16) return fail(MOA_ERR_INVALID_P, "p=%d must be a power of two <= 16", p);
    if (n / p < p)
        return fail(MOA_ERR_INVALID_P, "psize = n/p = %lld < p = %d violates psize >= m (P:289)",
                    (long long)(n / p), p);
    if (mode == MOA_MODE_LITERAL && p != 1)
        return fail(MOA_ERR_INVALID_P, "literal mode is single-GPU (p must be 1, got %d)", p);
    if (mode == MOA_MODE_EMULATED && p < 2) return fail(MOA_ERR_INVALID_P, "emulated mode needs p >= 2");
    const int64_t batch = (opt && opt->batch > 1) ? opt->batch : 1;
    if (opt && opt->batch < 0) return fail(MOA_ERR_INVALID_ARG, "batch %lld < 0", (long long)opt->batch);
    if (batch > 1 && (p != 1 || mode != MOA_MODE_LIFTED))
        return fail(MOA_ERR_INVALID_ARG, "batch > 1 needs p == 1 and the lifted mode");
    if (batch > 1 && (double)batch * (double)n > 8.0 * (double)((int64_t)1 << 32))
        return fail(MOA_ERR_INVALID_ARG, "batch * n = %.3g elements is beyond one GPU", (double)batch * n);
    const int exchange = (p > 1 && opt) ? opt->exchange : MOA_XCHG_NCCL;
    if (exchange < MOA_XCHG_NCCL || exchange > MOA_XCHG_P2P_EXTERNAL)
        return fail(MOA_ERR_INVALID_ARG, "unknown exchange %d", exchange);
    int rank = 0;
    if (p > 1 && mode != MOA_MODE_EMULATED) {
        if (exchange == MOA_XCHG_P2P_EXTERNAL) {
            rank = opt->rank;
            if (rank < 0 || rank >= p) return fail(MOA_ERR_INVALID_ARG, "rank %d outside [0, %d)", rank, p);
        } else {
            int wr = -1, ws = 0;
            if (dist_world(&wr, &ws) != MOA_OK || ws == 0)
                return fail(MOA_ERR_NO_DIST, "p=%d > 1 needs moa_dist_init first", p);
            if (ws != p) return fail(MOA_ERR_INVALID_P, "p=%d differs from the world size %d", p, ws);
            rank = wr;
        }
    }
    int rc0 = MOA_OK;
    moa_fft_plan_s *pl = new moa_fft_plan_s();
    pl->n = n;
    pl->t = ilog2(n);
    pl->p = p;
    pl->rank = rank;
    pl->sign = sign;
    pl->mode = mode;
    pl->batch = batch;
    pl->exchange = exchange;
    pl->M = n / p;
    CUDA_TRY(cudaGetDevice(&pl->device));
    if ((rc0 = resolve_lifting(pl, opt)) != MOA_OK) {
        delete pl;
        return rc0;
    }
    pl->chunks = 1;

    // ---- S1: twiddle tables (sign -1; sign +1 runs conj(FFT(conj x)))
    pl->hbits = (pl->t + 1) / 2;
    int64_t nlo = (int64_t)1 << pl->hbits, nhi = (int64_t)1 << (pl->t - pl->hbits);
    std::vector<double2> hlo(nlo), hhi(nhi), hf(FMAX);
    for (int64_t e = 0; e < nlo; ++e) hlo[e] = host_root((uint64_t)e, (uint64_t)n);
    for (int64_t e = 0; e < nhi; ++e) hhi[e] = host_root((uint64_t)e << pl->hbits, (uint64_t)n);
    for (int e = 0; e < FMAX; ++e) hf[e] = host_root((uint64_t)e, FMAX);
    int rc = MOA_OK;
    auto alloc = [&](double2 **ptr, int64_t elems) -> int {
        if (elems <= 0) return MOA_OK;
        cudaError_t e = cudaMalloc((void **)ptr, (size_t)elems * sizeof(double2));
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(MOA_ERR_OOM, "cudaMalloc(%lld bytes) failed: %s", (long long)(elems * 16),
                        cudaGetErrorString(e));
        }
        pl->workspace_bytes += elems * (int64_t)sizeof(double2);
        return MOA_OK;
    };
    if ((rc = alloc(&pl->tw_lo, nlo)) || (rc = alloc(&pl->tw_hi, nhi)) || (rc = alloc(&pl->tw_f, FMAX))) {
        free_plan(pl);
        return rc;
    }
    cudaError_t ce;
    if ((ce = cudaMemcpy(pl->tw_lo, hlo.data(), nlo * 16, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (ce = cudaMemcpy(pl->tw_hi, hhi.data(), nhi * 16, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (ce = cudaMemcpy(pl->tw_f, hf.data(), FMAX * 16, cudaMemcpyHostToDevice)) != cudaSuccess) {
        free_plan(pl);
        return fail(MOA_ERR_CUDA, "twiddle upload failed: %s", cudaGetErrorString(ce));
    }
    static bool prepared = false;
    if (!prepared) {
        if ((ce = prepare_pass_kernels()) != cudaSuccess) {
            free_plan(pl);
            return fail(MOA_ERR_CUDA, "kernel attribute setup failed: %s", cudaGetErrorString(ce));
        }
        prepared = true;
    }

    // ---- buffers and passes
    if (mode == MOA_MODE_LITERAL) {
        pl->work_elems = n;
    } else {
        pl->work_elems = pl->d > 1 ? pl->M * pl->batch : 0;
        if (p > 1) pl->send_elems = (mode == MOA_MODE_EMULATED) ? n : pl->M;
    }
    // P2P: no send buffer; real ranks double-buffer the receive buffer (one barrier per execute)
    const bool p2p = p > 1 && exchange != MOA_XCHG_NCCL;
    const int64_t recv_elems = p2p && mode != MOA_MODE_EMULATED ? 2 * pl->send_elems : pl->send_elems;
    if ((rc = alloc(&pl->work, pl->work_elems)) || (rc = alloc(&pl->send, p2p ? 0 : pl->send_elems)) ||
        (rc = alloc(&pl->recv, recv_elems))) {
        free_plan(pl);
        return rc;
    }
    if (mode == MOA_MODE_EMULATED) {
        pl->rank_passes.resize(p);
        for (int r = 0; r < p; ++r)
            if ((rc = build_passes(pl, r, p, pl->rank_passes[r])) != MOA_OK) {
                free_plan(pl);
                return rc;
            }
        for (auto &rp : pl->rank_passes)
            for (auto &pp : rp) choose_tma(pp);
    } else if (mode == MOA_MODE_LIFTED) {
        if ((rc = build_passes(pl, rank, p, pl->passes)) != MOA_OK) {
            free_plan(pl);
            return rc;
        }
        if (batch == 1)
            for (auto &pp : pl->passes) choose_tma(pp);
        const int fuse = batch == 1 ? env_int("MOA_FFT_FUSE", 0) : 0;
        if (p == 1 && pl->d == 3 && fuse && (rc = setup_fused(pl, fuse)) != MOA_OK) {
            free_plan(pl);
            return rc;
        }
    }
    *res = pl;
    return MOA_OK;
}

// Multi-dimensional transform of a row-major n_0 x ... x n_{r-1} array:
// App. B's Omega applies a 1-D operation to every sub-array along an axis (B.1-B.6,
// P:1495-1548), so the r-D DFT is the 1-D FFT applied along each axis in turn.
// Last axis: a batched lifted 1-D plan (batch = product of the other extents, any
// length).  Every other axis a: ONE pass of n_a-point DFTs along the stride
// B = n_{a+1}...n_{r-1} axis -- the middle-pass tile of §4 with the view
// [A = n_0...n_{a-1}][n_a][B], T adjacent columns per tile, no twiddle, in place --
// so n_a <= FMAX for a < r-1.
static int make_plan_nd(int rank, const int64_t *shape, int sign, moa_fft_plan_s **res) {
    *res = nullptr;
    if (rank < 2 || rank > 3) return fail(MOA_ERR_INVALID_ARG, "rank %d must be 2 or 3", rank);
    if (sign != -1 && sign != 1) return fail(MOA_ERR_INVALID_SIGN, "sign=%d must be -1 or +1", sign);
    int64_t total = 1;
    for (int a = 0; a < rank; ++a) {
        const int64_t na = shape[a];
        if (!pow2(na) || na < 2 || (a < rank - 1 && na > (int64_t)FMAX * FMAX))
            return fail(MOA_ERR_INVALID_N, "n%d=%lld must be 2^t with 1 <= t%s", a + 1, (long long)na,
                        a < rank - 1 ? " <= 26 (at most two passes along a non-last axis)" : "");
        total *= na;
        if (total > ((int64_t)1 << 32))
            return fail(MOA_ERR_INVALID_N, "the array holds more than 2^32 elements");
    }
    moa_fft_options o;
    memset(&o, 0, sizeof o);
    o.mode = MOA_MODE_LIFTED;
    o.batch = total / shape[rank - 1];
    moa_fft_plan_s *rows = nullptr;
    int rc = make_plan(shape[rank - 1], 1, sign, &o, &rows);
    if (rc) return rc;
    moa_fft_plan_s *pl = new moa_fft_plan_s();
    pl->rows = rows;
    pl->n1 = shape[0];
    pl->n2 = total / shape[0];
    pl->n = total;
    pl->M = total;
    pl->t = ilog2(total);
    pl->sign = sign;
    pl->device = rows->device;
    pl->d = rank - 1;
    auto axis_pass = [&](int logF, int64_t B) {
        PassPlan pp;
        memset(&pp.d, 0, sizeof(PassDesc));
        pp.logF = logF;
        pp.T = choose_T(logF, B);
        PassDesc &D = pp.d;
        D.hbits = rows->hbits;
        D.tw_hi = rows->tw_hi;
        D.tw_lo = rows->tw_lo;
        D.tw_f = rows->tw_f;
        D.pack_lp = -1;
        D.in_t = 1;
        D.out_t = 1;
        D.in_tfast = D.out_tfast = pp.T > 1;
        D.U = B / pp.T;
        D.lU = ilog2(D.U);
        D.in_u = D.out_u = pp.T;
        return pp;
    };
    bool need_work = false;
    for (int a = rank - 2; a >= 0; --a) {   // execution order: the last-but-one axis first
        int64_t A = 1, B = 1;
        for (int l = 0; l < a; ++l) A *= shape[l];
        for (int l = a + 1; l < rank; ++l) B *= shape[l];
        const int64_t N = shape[a];
        if (N <= FMAX) {   // one pass, in place: view [A][N][B]
            PassPlan pp = axis_pass(ilog2(N), B);
            PassDesc &D = pp.d;
            D.nmask = (uint64_t)N - 1;
            D.tbits = pp.logF;
            D.conj_in = D.conj_out = sign > 0;   // conj(DFT_-1(conj y)) along this axis
            D.V = A;
            D.lV = ilog2(D.V);
            D.in_v = D.out_v = N * B;
            D.in_f = D.out_k = B;
            pp.tiles = D.U * D.V;
            pl->passes.push_back(pp);
        } else {
            // a lifted strided axis, N = N1 * N2 (the reshape-transpose of §4 along axis a):
            // element (alpha, j1, j2, beta) at ((alpha*N1 + j1)*N2 + j2)*B + beta.
            //   pass A (out -> work): N1-point DFTs over j1 (stride N2*B), times omega_N^(j2*k1)
            //   pass B (work -> out): N2-point DFTs over j2 (stride B), stored at
            //                         (alpha*N + k1 + N1*k2)*B + beta (the transposed store)
            const int tN = ilog2(N), t1 = tN / 2, t2 = tN - t1;
            const int64_t N1 = (int64_t)1 << t1, N2 = (int64_t)1 << t2;
            const int hb = (tN + 1) / 2;
            const int64_t nlo = (int64_t)1 << hb, nhi = (int64_t)1 << (tN - hb);
            std::vector<double2> hlo(nlo), hhi(nhi);
            for (int64_t e = 0; e < nlo; ++e) hlo[e] = host_root((uint64_t)e, (uint64_t)N);
            for (int64_t e = 0; e < nhi; ++e) hhi[e] = host_root((uint64_t)e << hb, (uint64_t)N);
            double2 *dlo = nullptr, *dhi = nullptr;
            if (cudaMalloc((void **)&dlo, nlo * 16) != cudaSuccess || cudaMalloc((void **)&dhi, nhi * 16) != cudaSuccess) {
                cudaGetLastError();
                cudaFree(dlo);
                free_plan(pl);
                return fail(MOA_ERR_OOM, "axis twiddle tables");
            }
            pl->axis_tw.push_back(dlo);
            pl->axis_tw.push_back(dhi);
            if (cudaMemcpy(dlo, hlo.data(), nlo * 16, cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(dhi, hhi.data(), nhi * 16, cudaMemcpyHostToDevice) != cudaSuccess) {
                free_plan(pl);
                return fail(MOA_ERR_CUDA, "axis twiddle upload failed");
            }
            PassPlan pa = axis_pass(t1, B);
            {
                PassDesc &D = pa.d;
                D.nmask = (uint64_t)N - 1;
                D.tbits = tN;
                D.hbits = hb;
                D.tw_hi = dhi;
                D.tw_lo = dlo;
                D.conj_in = sign > 0;
                D.twiddle = 1;
                D.b_v = 1;   // exponent j2 * k1 (v = j2)
                D.V = N2;
                D.lV = t2;
                D.in_v = D.out_v = B;
                D.in_w = D.out_w = N * B;
                D.in_f = D.out_k = N2 * B;
                pa.tiles = D.U * D.V * A;
                pa.io = 1;
            }
            PassPlan pb = axis_pass(t2, B);
            {
                PassDesc &D = pb.d;
                D.nmask = (uint64_t)N - 1;
                D.tbits = tN;
                D.conj_out = sign > 0;
                D.V = N1;
                D.lV = t1;
                D.in_v = N2 * B;
                D.in_w = N * B;
                D.in_f = B;
                D.out_v = B;
                D.out_w = N * B;
                D.out_k = N1 * B;
                pb.tiles = D.U * D.V * A;
                pb.io = 2;
            }
            if (!pass_supported(pa.logF, pa.T) || !pass_supported(pb.logF, pb.T)) {
                free_plan(pl);
                return fail(MOA_ERR_INVALID_ARG, "no pass kernel for an axis of length 2^%d", tN);
            }
            pl->passes.push_back(pa);
            pl->passes.push_back(pb);
            need_work = true;
        }
        if (a + 1 < 4) pl->lift[a + 1] = N;
    }
    for (const PassPlan &pp : pl->passes)
        if (!pass_supported(pp.logF, pp.T)) {
            free_plan(pl);
            return fail(MOA_ERR_INVALID_ARG, "no pass kernel for F=2^%d T=%d", pp.logF, pp.T);
        }
    if (need_work) {
        if (cudaMalloc((void **)&pl->work, (size_t)total * sizeof(double2)) != cudaSuccess) {
            cudaGetLastError();
            free_plan(pl);
            return fail(MOA_ERR_OOM, "r-D work buffer (%lld elements)", (long long)total);
        }
        pl->work_elems = total;
        pl->workspace_bytes += total * 16;
    }
    pl->lift[0] = shape[rank - 1];
    pl->stream = rows->stream;
    *res = pl;
    return MOA_OK;
}

static bool aligned16(const void *ptr) { return ptr && ((uintptr_t)ptr & 15) == 0; }

// ---- event profiling: a scope records an event pair around one launch
static cudaEvent_t pool_event(moa_fft_plan_s *pl) {
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
static int launch_pp(moa_fft_plan_s *pl, PassPlan &pp, int idx, const double2 *src, double2 *dst,
                     double2 *const *peers = nullptr, int64_t peer_off = 0) {
    PassDesc D = pp.d;
    D.src = src;
    D.dst = dst;
    if (peers) {
        for (int r = 0; r < pl->p; ++r) D.peer[r] = peers[r];
        D.peer_off = peer_off;
    }
    char name[64];
    snprintf(name, sizeof name, "pass%d fft_pass%s<F=%d,T=%d>%s", idx, pp.tma ? "_tma" : (pp.pf_grid ? "_pf" : ""),
             1 << pp.logF, pp.T,
             peers ? "+push" : "");
    ProfScope ps_(pl, name, 32 * pl->M * pl->batch);
    cudaError_t e;
    if (pp.tma && !peers) {
        if (pp.map_base != (const void *)src) {
            int rc = encode_pass_map(pp, src);
            if (rc) return rc;
        }
        e = launch_pass_tma(pp.logF, pp.T, pp.tma, D, pp.map, pp.tiles, pp.tma_grid, pl->stream);
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
static int run_passes(moa_fft_plan_s *pl, std::vector<PassPlan> &ps, const double2 *in, double2 *out,
                      double2 *const *peers = nullptr, int64_t peer_off = 0) {
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
static int p2p_phase(moa_fft_plan_s *pl, const double2 *in, double2 *out, int phase) {
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

static int execute(moa_fft_plan_s *pl, const double2 *in, double2 *out) {
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

}  // namespace moa

// ====================================================================== C ABI
extern "C" {

moa_fft_plan_t moa_fft_plan_ex(int64_t n, int p, int sign, const moa_fft_options *opts) {
    g_err.clear();
    moa_fft_plan_s *pl = nullptr;
    if (make_plan(n, p, sign, opts, &pl) != MOA_OK) return nullptr;
    return pl;
}

moa_fft_plan_t moa_fft_plan(int64_t n, int p, int sign) { return moa_fft_plan_ex(n, p, sign, nullptr); }

moa_fft_plan_t moa_fft_plan_nd(int rank, const int64_t *shape, int sign) {
    g_err.clear();
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
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != pl->device) cudaSetDevice(pl->device);
    int rc = execute(pl, (const double2 *)in, (double2 *)out);
    if (cur != pl->device) cudaSetDevice(cur);
    return rc;
}

int moa_fft_execute_host(moa_fft_plan_t pl, const void *host_in, void *host_out) {
    if (!pl) return fail(MOA_ERR_INVALID_ARG, "NULL plan");
    if (!host_in || !host_out) return fail(MOA_ERR_ALIGN, "NULL host buffer");
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
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != pl->device) cudaSetDevice(pl->device);
    struct Restore {
        int cur, dev;
        ~Restore() {
            if (cur != dev) cudaSetDevice(cur);
        }
    } restore_{cur, pl->device};
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
    o->breakpoint = ilog2(pl->M) + 1;
    o->chunks = pl->chunks;
    if (pl->mode == MOA_MODE_LITERAL) {
        o->launches = pl->t + 1;
        o->hbm_bytes = 32 * pl->n * (pl->t + 1);
    } else if (pl->p == 1) {
        o->launches = pl->fused ? pl->d - 1 : pl->d;
        o->hbm_bytes = 32 * pl->n * pl->batch * (pl->fused ? pl->d - 1 : pl->d);
    } else {
        int per_rank = pl->d + 1;
        o->launches = pl->mode == MOA_MODE_EMULATED ? pl->p * per_rank : per_rank;
        o->hbm_bytes = 32 * pl->M * (pl->d + 1) * (pl->mode == MOA_MODE_EMULATED ? pl->p : 1);
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

const char *moa_fft_last_error(void) { return g_err.c_str(); }

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
    int rc = resolve_lifting(&tmp, opts);
    if (rc) return rc;
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
