// plan.cu -- the plan builder: S0 validation and dimension lifting, S1 twiddle
// tables, the per-pass index maps (PassDesc), the L2-fused and TMA variants, and
// the r-D plans.
//
//   S0 validation and lifting   n = 2^t, psize = n/p >= p, breakpoint =
//                               log2(psize)+1 (the high end of §4.8)
//   S1 twiddle tables           built once per plan in long double (the paper
//                               recomputes weight(row) every stage)
//   S3/S4 lifted passes         one PassDesc per level of <F1..Fd>
//   S5/S6 (p > 1)               the local psize-point FFT whose last pass scales by
//                               omega_n^(r*k1) and routes to the destination ranks (Fig 5.9)
// The executor is exec.cu, the C ABI abi.cu.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "plan_internal.h"

namespace moa {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static thread_local int g_code = MOA_OK;

void clear_error() {
    g_err.clear();
    g_code = MOA_OK;
}
const char *last_error() { return g_err.c_str(); }
int last_error_code() { return g_code; }

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    g_code = code;
    return code;
}

// ------------------------------------------------------------------ twiddles
// exp(-2 pi i e / N) for N a power of two, evaluated in long double on the
// first octant of the circle and rounded once to double; quarter turns exact.
double2 host_root(uint64_t e, uint64_t N) {
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


// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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
int encode_pass_map(PassPlan &pp, const void *base) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return fail(MOA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const PassDesc &D = pp.d;
    const uint64_t F = 1ull << pp.logF, T = pp.T;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
    cuuint32_t rank;
    if (pp.tma == 1 || pp.tma == 4 || pp.tma == 6 || (pp.big && !pp.d.last)) {   // column tile of the view [A][F][B]: dims {2B doubles, F, A}
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

// output map of a bulk-tensor-store last pass: dims {2*K_k doubles (inner index), F (k)}
int encode_out_map(PassPlan &pp, const void *base) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return fail(MOA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const PassDesc &D = pp.d;
    const uint64_t F = 1ull << pp.logF, T = pp.T, Kk = (uint64_t)D.K_k;
    cuuint64_t dims[2] = {2 * Kk, F}, strides[1] = {16 * Kk};
    cuuint32_t box[2] = {(cuuint32_t)(2 * T), (cuuint32_t)(F < 256 ? F : 256)}, estr[2] = {1, 1};
    CUresult r = enc(&pp.omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(MOA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for the output map", (int)r);
    pp.omap_base = base;
    return MOA_OK;
}

// choose the TMA-staged variant when it exists for this (F, T, layout), else the
// prefetching persistent kernel when selected
void choose_tma(PassPlan &pp) {
    pp.tma = 0;
    pp.pf_grid = 0;
#ifndef MOA_VARIANTS
    (void)pp;
    return;   // the persistent / TMA-staged variants live in libmoa_fft_variants.so only
#else
    const int pf_env = env_int("MOA_FFT_PF", 0);
    if (pf_env && pp.logF >= 5) {
        int g = pass_pf_grid(pp.logF, pp.T);
        if (g > 0) pp.pf_grid = (int)(g < pp.tiles ? g : pp.tiles);
    }
    const int tma_kind = env_int("MOA_FFT_TMA", 0);   // 1: double-buffered TMA, 2: single buffer + prefetch
    if (tma_kind == 0) return;
    const PassDesc &D = pp.d;
    int src = 0;
    if (!D.last && D.in_t == 1 && pp.T >= 2) src = 1;
    else if (D.last && D.in_f == 1) src = 2;
    if (!src) return;
    // 1: persistent double-buffered, 2: persistent single buffer + prefetch (src 4/5),
    // 3: one tile per CTA loaded by one bulk-tensor copy (src 6/7, fft_pass_tma1_kernel)
    const int code = tma_kind == 2 ? src + 3 : (tma_kind == 3 ? src + 5 : src);
    int g = pass_tma_grid(pp.logF, pp.T, code);
    if (g <= 0) return;
    pp.tma = code;
    pp.tma_grid = code >= 6 ? (int)pp.tiles : g;
#endif
}

// default lifting <F1..Fd> of a local length 2^tl, from the B200 lifting sweeps
// (tools/perf_probe.py): 256-point passes (4 tiles per SM) wherever the
// length allows, the remaining factor in the row pass up to 2^12, four levels from 2^29
// on (two <= 128-point column passes instead of one long one).  p > 1 plans keep <= 3
// levels.
int default_lifting(int tl, int64_t *lift, int p) {
    if (tl <= 12) {   // one CTA per transform (2^13 in one CTA: 18.4 us, as <64,128>: 12.3 us)
        lift[0] = (int64_t)1 << tl;
        return 1;
    }
    if (p == 1 && (tl == 15 || tl == 20)) {   // <256, 128> and <256, 4096>: 8.1 vs 9.7 us as <128, 256>,
        lift[0] = 256;                         // 22.1 vs 24.2 us as <1024, 1024> (L2-flushed, batched
        lift[1] = (int64_t)1 << (tl - 8);      // event timing, tools/tune_probe.py)
        return 2;
    }
    if (tl <= 20) {   // two levels, the longer one last: <256,256> at 2^16, <512,1024> at 2^19
        int a = tl / 2;
        lift[0] = (int64_t)1 << a;
        lift[1] = (int64_t)1 << (tl - a);
        return 2;
    }
    if (tl == 21 || tl == 22) {   // <128, 256, 2^(tl-15)>: 2^21 38.9 vs 47.1 us as <32,256,256>,
        lift[0] = 128;               // 2^22 69.7 vs 73.8 us as <64,256,256> (tools/tune_probe.py):
        lift[1] = 256;               // a <= 64-point first pass (T >= 32) is the slowest of the three
        lift[2] = (int64_t)1 << (tl - 15);
        return 3;
    }
    if (tl >= 25 && tl <= 28) {   // <256, 256, 2^(tl-16)>: the long factor in the row pass
        lift[0] = 256;
        lift[1] = 256;
        lift[2] = (int64_t)1 << (tl - 16);
        return 3;
    }
    if (p > 1 && tl == 29) {   // <256, 512, 4096> (p > 1 keeps <= 3 levels): per rank of 2^30 over
        lift[0] = 256;         // 2 virtual ranks 13.7 ms vs 21.0 ms as <8192, 256, 256>, 14.0 as
        lift[1] = 512;         // <512, 256, 4096>, 15.1 as <512, 512, 2048> (tools/lift_p_probe.py)
        lift[2] = 4096;
        return 3;
    }
    if (p > 1 && tl == 30) {   // <512, 512, 4096>: per rank of 2^31 over 2 virtual ranks 30.3 ms vs
        lift[0] = 512;         // 32.8 as <1024, 1024, 1024>, 30.6 as <256, 1024, 4096>
        lift[1] = 512;
        lift[2] = 4096;
        return 3;
    }
    if (tl <= 27 || (p > 1 && tl <= 16 + FMAX_LOG)) {   // <2^(tl-16), 256, 256>
        lift[0] = (int64_t)1 << (tl - 16);
        lift[1] = 256;
        lift[2] = 256;
        return 3;
    }
    if (tl == 29 && p == 1) {   // <128, 128, 128, 256>: 10.60 vs 11.31 ms as <64, 128, 256, 256>
        lift[0] = 128;           // (a 64-point first pass of T = 32 was the slowest of the four)
        lift[1] = 128;
        lift[2] = 128;
        lift[3] = 256;
        return 4;
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

int choose_T(int logF, int64_t avail) {
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

// Small transforms: halve T while the pass would have fewer than ~one tile per SM
// (measured: 2^18 <512,512> 18.5 -> 16.4 us), keeping T >= 2 for the column runs.
static int fill_T(int T, int64_t transforms, int64_t batch) {
    const int64_t min_tiles = env_int("MOA_FFT_MINTILES", 128);
    while (T > 2 && transforms * batch / T < min_tiles) T /= 2;
    return T;
}

// Build the passes of a local FFT of length M = prod(lift) (global length n).
// rank >= 0 with P > 1: the last pass scales by omega_n^(rank*K) and packs to
// the send layout [dst][c] with K = dst + P*c (S6, fused into S4's epilogue).
int build_passes(const moa_fft_plan_s *pl, int rank, int P, std::vector<PassPlan> &out) {
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
            int T = fill_T(choose_T(pp.logF, B), pl->M / F, pl->batch);
            // first column pass over rows >= 1 MiB apart: 256-byte runs (T*F = 4096, 2 tiles
            // per SM) -- each 128-byte run of a T = 8 tile opens its own DRAM page (F = 256
            // only: 64- and 128-point first passes of 2^29 / 2^30 lose 2-3 % at T = 64 / 32)
            if (i == 0 && pp.logF == 8 && (int64_t)16 * B >= env_int("MOA_FFT_WIDE", 1 << 20) &&
                T == (2048 >> pp.logF) && 2 * T <= B && pass_supported(pp.logF, 2 * T) && pl->batch == 1)
                T *= 2;
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
                int T = fill_T(choose_T(pp.logF, Fv[0]), pl->M / F, pl->batch);
                // with bulk-tensor stores (make_plan: MOA_FFT_TMAST) the 512- and 1024-point row
                // passes take 2048-element tiles (4 CTAs/SM): the TMA engine scatters their
                // 64- / 32-byte runs (2^25 F = 512 190 -> 175 us, 2^26 F = 1024 384 -> 355 us)
                if (P == 1 && pl->batch == 1 && pl->M >= ((int64_t)1 << 22) && (pp.logF == 9 || pp.logF == 10) &&
                    env_int("MOA_FFT_TMAST", 9) > 0 && env_int("MOA_FFT_TMAST", 9) <= pp.logF &&
                    (T << pp.logF) > 2048 && pass_supported(pp.logF, 2048 >> pp.logF))
                    T = 2048 >> pp.logF;
                // 256-byte output runs (T = 16, 2 tiles per SM) when the transposed store's
                // rows are >= 1 MiB apart (MOA_FFT_WIDE_LAST, bytes; 0 = off): 2^24 pass 2
                // 91.4 -> 90.4 us, step 258.6 -> 256.8 us (bench, 3 alternating runs)
                {
                    const int wl = env_int("MOA_FFT_WIDE_LAST", 1 << 20);
                    if (wl > 0 && P == 1 && pp.logF == 8 && (int64_t)16 * Kk >= wl && T == (2048 >> pp.logF) &&
                        2 * T <= Fv[0] && pass_supported(pp.logF, 2 * T) && pl->batch == 1)
                        T *= 2;
                }
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
        // ablation (libmoa_fft_variants.so, MOA_FFT_BIG=1): 4096-point passes of T = 2 as the
        // persistent TMA-fed kernel (bigpass.cu) -- single-GPU, unbatched plans whose column
        // tiles are plain [A][F][B] views and whose row tiles are contiguous rows.  Measured
        // slower than three 256-point passes at 2^24, so never the default.
        if (P == 1 && pl->batch == 1 && big_supported(pp.logF, pp.T) && pp.tiles >= 2 &&
            env_int("MOA_FFT_BIG", 0) && D.in_shift == 0 && D.out_shift == 0 && D.pack_lp < 0 &&
            (D.last ? D.in_f == 1 : (D.in_t == 1 && D.in_w == 0 && D.in_u == pp.T)))
            pp.big = 1;
        out.push_back(pp);
    }
    return MOA_OK;
}

// SURVEY §8(e) chunked exchange: the last pass of a 3-level p > 1 lifting split into G
// groups of its middle digit w (k_1).  Group g writes its outputs, for every
// destination, into send chunk g in the layout [g][dst][o][i] with
// o = w_local + (F1/G)*k and i = T*u + t, so the all-to-all of chunk g can start while
// group g+1 is being computed; pcombine_chunk maps the received chunk back to columns.
int build_chunked_last(const moa_fft_plan_s *pl, const PassPlan &last, int G, std::vector<PassPlan> &out) {
    out.clear();
    const int64_t F0 = pl->lift[0], F1 = pl->lift[1], M = pl->M, P = pl->p;
    if (pl->d != 3 || G < 2 || F1 % G) return fail(MOA_ERR_INVALID_ARG, "chunks=%d needs a 3-level lifting with G | F1", G);
    const int64_t Wg = F1 / G;
    for (int g = 0; g < G; ++g) {
        PassPlan pp = last;
        PassDesc &D = pp.d;
        D.pack_lp = -1;
        D.in_shift = -(int64_t)g * Wg * D.in_w;                   // w = g*Wg + w_local
        D.a_c = (int64_t)((uint64_t)D.a_c + (uint64_t)D.a_w * (uint64_t)(g * Wg));
        D.out_shift = -(int64_t)g * (M / G);                      // chunk g of the send buffer
        D.out_v = M / (G * P);                                    // destination block inside the chunk
        D.out_u = pp.T;
        D.out_t = 1;
        D.out_w = F0 / P;
        D.out_k = Wg * (F0 / P);
        pp.tiles = D.U * D.V * Wg;
        pp.tma = 0;
        pp.pf_grid = 0;
        out.push_back(pp);
    }
    return MOA_OK;
}

void free_plan(moa_fft_plan_s *pl) {
    if (!pl) return;
    if (pl->lowsub) {
        free_plan(pl->lowsub);
        pl->lowsub = nullptr;
    }
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
    if (pl->comm_stream) cudaStreamDestroy(pl->comm_stream);
    if (pl->comb_stream) cudaStreamDestroy(pl->comb_stream);
    for (cudaEvent_t e : pl->ev_pass)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : pl->ev_a2a)
        if (e) cudaEventDestroy(e);
    if (pl->ev_comb) cudaEventDestroy(pl->ev_comb);
    if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
    if (pl->graph_stream) cudaStreamDestroy(pl->graph_stream);
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
int setup_fused(moa_fft_plan_s *pl, int kind) {
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
int resolve_lifting(moa_fft_plan_s *pl, const moa_fft_options *opt) {
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

int resolve_breakpoint(moa_fft_plan_s *pl, const moa_fft_options *opt) {
    const int bp = opt ? opt->breakpoint : 0;
    const int lm = ilog2(pl->p), lps = ilog2(pl->M);
    pl->lowend = false;
    if (bp == 0 || bp == lps + 1) return MOA_OK;
    if (pl->p > 1 && bp == lm + 1) {
        if (pl->M < 2 * (int64_t)pl->p)
            return fail(MOA_ERR_INVALID_ARG, "low-end breakpoint needs n/p >= 2p (psize = %lld, p = %d)",
                        (long long)pl->M, pl->p);
        pl->lowend = true;
        return MOA_OK;
    }
    return fail(MOA_ERR_INVALID_ARG,
                "breakpoint %d: the GPU path runs the high end %d (P:289) or, for p > 1, the low end %d (P:694)", bp,
                lps + 1, lm + 1);
}

int make_plan(int64_t n, int p, int sign, const moa_fft_options *opt, moa_fft_plan_s **res) {
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
    if ((rc0 = resolve_breakpoint(pl, opt)) != MOA_OK) {
        delete pl;
        return rc0;
    }
    if (pl->lowend) {
        // low-end breakpoint (Fig 5.7, breakpoint = log2 m + 1).  Rank u receives
        // W[j''] for j'' = r + P*c in [source r][c] blocks and needs X[u + P*v] =
        // sum_j'' omega_M^(j''*v) W[j''].  With v = v1 + (M/P)*v2:
        //   X = sum_r omega_P^(r*v2) * omega_M^(r*v1) * [sum_c omega_{M/P}^(c*v1) W[r][c]]
        // -- P contiguous (M/P)-point FFTs (a batched p = 1 plan; options.lift is ITS
        // lifting), then pcombine with the omega_M^(r*v1) factor on its loads.
        moa_fft_options so = {};
        so.mode = MOA_MODE_LIFTED;
        so.batch = p;
        if (opt && opt->nlift > 0) {
            so.nlift = opt->nlift;
            for (int i = 0; i < opt->nlift && i < 4; ++i) so.lift[i] = opt->lift[i];
        }
        if (exchange != MOA_XCHG_NCCL) {   // (checked before the sub-plan owns device memory)
            delete pl;
            return fail(MOA_ERR_INVALID_ARG, "the low-end breakpoint runs with the NCCL exchange (or EMULATED ranks)");
        }
        if ((rc0 = make_plan(pl->M / p, 1, -1, &so, &pl->lowsub)) != MOA_OK) {
            delete pl;
            return rc0;
        }
        pl->d = pl->lowsub->d;
        for (int i = 0; i < 4; ++i) pl->lift[i] = pl->lowsub->lift[i];
    } else if ((rc0 = resolve_lifting(pl, opt)) != MOA_OK) {
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
    {
        // the dynamic shared-memory limits are per-device function attributes: raise them
        // once for every device a plan is built on (serialised across threads)
        static std::mutex mu;
        static uint64_t prepared_mask = 0;
        std::lock_guard<std::mutex> lock(mu);
        const uint64_t bit = 1ull << (pl->device & 63);
        if (!(prepared_mask & bit)) {
            if ((ce = prepare_pass_kernels()) != cudaSuccess) {
                free_plan(pl);
                return fail(MOA_ERR_CUDA, "kernel attribute setup failed: %s", cudaGetErrorString(ce));
            }
            prepared_mask |= bit;
        }
    }

    // ---- buffers and passes
    if (mode == MOA_MODE_LITERAL) {
        pl->work_elems = n;
    } else {
        pl->work_elems = (pl->d > 1 || pl->lowend) ? pl->M * pl->batch : 0;
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
    if (pl->lowend) {
        // no passes of its own: psplit, the exchange, lowsub, pcombine (exec.cu)
    } else if (mode == MOA_MODE_EMULATED) {
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
        // bulk-tensor stores for the row pass from F = 512 on (MOA_FFT_TMAST = minimum log2 F,
        // 0 = off): the per-lane transposed stores of T <= 4 rows throttle the LSU; measured
        // 2^26 F = 1024 403 -> 384 us (T = 4; 355 us at T = 2), 2^27 F = 2048 964 -> 841 us,
        // 2^28 F = 4096 2345 -> 2323 us; slower at F = 256 (90.5 -> 102, T = 16) and at
        // F = 512 with T = 8 (190 -> 194; T = 4 gives 175)
        const int tmast_min = env_int("MOA_FFT_TMAST", 9);
        if (p == 1 && batch == 1 && tmast_min > 0 && pl->M >= ((int64_t)1 << 22) && !pl->passes.empty()) {
            // (HBM-sized transforms only: at 2^19 / 2^20 it measured equal or slower)
            PassPlan &lp = pl->passes.back();
            const PassDesc &D = lp.d;
            if (D.last && lp.logF >= tmast_min && lp.logF >= 8 && !lp.tma && !lp.pf_grid && D.pack_lp < 0 &&
                D.K_t == 1 && D.out_t == 1 && D.out_k == D.K_k && D.out_u == D.K_u && D.out_v == D.K_v &&
                D.out_w == D.K_w && 2 * lp.T <= 256)
                lp.tmast = 1;
        }
        const int fuse = batch == 1 ? env_int("MOA_FFT_FUSE", 0) : 0;
        if (p == 1 && pl->d == 3 && fuse && (rc = setup_fused(pl, fuse)) != MOA_OK) {
            free_plan(pl);
            return rc;
        }
    }
    // chunked NCCL exchange: G groups of the last pass's middle digit,
    // each all-to-all overlapping the next group's butterflies.  Default G: per-peer
    // chunks of >= 1 MiB, at most 8 (real ranks); EMULATED plans chunk only when asked.
    if (opt && opt->chunks > 1 && !(p > 1 && exchange == MOA_XCHG_NCCL && pl->d == 3 && !pl->lowend)) {
        free_plan(pl);
        return fail(MOA_ERR_INVALID_ARG, "chunks=%d needs p > 1, the NCCL exchange and a 3-level lifting", opt->chunks);
    }
    if (p > 1 && exchange == MOA_XCHG_NCCL && mode != MOA_MODE_LITERAL && pl->d == 3 && !pl->lowend) {
        int G = opt && opt->chunks > 0 ? opt->chunks : 0;
        if (G == 0 && mode == MOA_MODE_LIFTED) {
            G = 1;
            while (G < 8 && (pl->M / (2 * G * p)) * 16 >= ((int64_t)1 << 20) && pl->lift[1] % (2 * G) == 0) G *= 2;
        }
        if (G > 1) {
            if (!pow2(G) || pl->lift[1] % G) {
                free_plan(pl);
                return fail(MOA_ERR_INVALID_ARG, "chunks=%d must be a power of two dividing F1=%lld", G,
                            (long long)pl->lift[1]);
            }
            if (mode == MOA_MODE_EMULATED) {
                pl->rank_chunk_last.resize(p);
                for (int r = 0; r < p; ++r)
                    if ((rc = build_chunked_last(pl, pl->rank_passes[r].back(), G, pl->rank_chunk_last[r])) != MOA_OK) {
                        free_plan(pl);
                        return rc;
                    }
            } else if ((rc = build_chunked_last(pl, pl->passes.back(), G, pl->chunk_last)) != MOA_OK) {
                free_plan(pl);
                return rc;
            }
            pl->ev_pass.resize(G);
            pl->ev_a2a.resize(G);
            bool ok = cudaStreamCreateWithFlags(&pl->comm_stream, cudaStreamNonBlocking) == cudaSuccess &&
                      cudaStreamCreateWithFlags(&pl->comb_stream, cudaStreamNonBlocking) == cudaSuccess &&
                      cudaEventCreateWithFlags(&pl->ev_comb, cudaEventDisableTiming) == cudaSuccess;
            for (int g = 0; ok && g < G; ++g)
                ok = cudaEventCreateWithFlags(&pl->ev_pass[g], cudaEventDisableTiming) == cudaSuccess &&
                     cudaEventCreateWithFlags(&pl->ev_a2a[g], cudaEventDisableTiming) == cudaSuccess;
            if (!ok) {
                cudaGetLastError();
                free_plan(pl);
                return fail(MOA_ERR_CUDA, "chunk streams/events creation failed");
            }
            pl->chunks = G;
        }
    }
    // graph replay: single-GPU lifted plans whose launches do not change between
    // executes (the fused kernel's epoch counter does; p > 1 alternates buffers)
    // (measured: 2^14-2^18 -1 us, 2^24 271.4 -> 268.3 us; a one-kernel plan gains nothing)
    pl->graph_ok = p == 1 && mode == MOA_MODE_LIFTED && !pl->fused && pl->d >= 2 && env_int("MOA_FFT_GRAPH", 1);
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
int make_plan_nd(int rank, const int64_t *shape, int sign, moa_fft_plan_s **res) {
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
        // one in-place pass while its column tiles keep >= 64-byte runs (T >= 4); longer
        // axes as two lifted passes (2-D 4096 x 4096: columns 205 -> 2 x ~87 us; 8192 x 8192:
        // one T = 1 pass of 16-byte runs took 1216 us, tools/nd_probe.py)
        if (N <= 1024) {   // one pass, in place: view [A][N][B]
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

}  // namespace moa
