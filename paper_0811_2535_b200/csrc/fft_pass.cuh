// fft_pass.cuh -- the lifted butterfly pass kernel.
//
// One CTA owns a tile of T independent F-point transforms (F = 2^f <= 8192)
// that lie along one lifted axis of the data (the reshape that
// "lifts" n into <F1, ..., Fd>).  Inside the CTA the F-point transform is the
// paper's radix-2 butterfly network (Fig 3.7 basic block) grouped
// into radix-16 register kernels: each thread holds 16 points, does
// log2(16) = 4 radix-2 butterfly levels in registers, and the levels between
// register kernels exchange data through shared memory in Stockham
// (self-sorting) order, so no separate bit-reversal pass is needed (P_n,
// P:105, is absorbed: the lifted index maps below place every output).
//
// Data movement per CTA: one read of T*F complex128 from global memory, one
// write, ceil(f/4) - 1 shared-memory exchanges.  The global-facing stages
// assign lanes so that consecutive lanes touch consecutive addresses
// (T-fastest for column tiles, j-fastest for row tiles).
//
// All arithmetic is for sign -1; sign +1 is conj(FFT(conj x)) (conj_in /
// conj_out flags), so every table is the omega^-e table.
#pragma once
#include "moa_internal.h"
#include "tma.cuh"

namespace moa {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// a * omega_16^k = a * exp(-2 pi i k / 16); k is a compile-time constant after unrolling.
__device__ __forceinline__ double2 mulw16(double2 a, int k) {
    const double C1 = 0.92387953251128675613;  // cos(pi/8)
    const double S1 = 0.38268343236508977173;  // sin(pi/8)
    const double C2 = 0.70710678118654752440;  // cos(pi/4)
    switch (k & 15) {
    case 0: return a;
    case 1: return cmul(a, make_double2(C1, -S1));
    case 2: return make_double2((a.x + a.y) * C2, (a.y - a.x) * C2);
    case 3: return cmul(a, make_double2(S1, -C1));
    case 4: return make_double2(a.y, -a.x);
    case 5: return cmul(a, make_double2(-S1, -C1));
    case 6: return make_double2((a.y - a.x) * C2, -(a.x + a.y) * C2);
    case 7: return cmul(a, make_double2(-C1, -S1));
    case 8: return make_double2(-a.x, -a.y);
    case 9: return cmul(a, make_double2(-C1, S1));
    case 10: return make_double2(-(a.x + a.y) * C2, (a.x - a.y) * C2);
    case 11: return cmul(a, make_double2(-S1, C1));
    case 12: return make_double2(-a.y, a.x);
    case 13: return cmul(a, make_double2(S1, C1));
    case 14: return make_double2((a.x - a.y) * C2, (a.x + a.y) * C2);
    default: return cmul(a, make_double2(C1, S1));
    }
}

template <int R>
__host__ __device__ constexpr int brev_c(int k) {
    int r = 0;
    for (int m = R >> 1, b = 1; m > 0; m >>= 1, b <<= 1)
        if (k & m) r |= b;
    return r;
}

// In-register R-point DFT (R = 2, 4, 8, 16), natural order in and out:
// log2 R levels of the radix-2 butterfly (decimation in frequency), then the
// compile-time bit-reversal renaming of registers (free).
template <int R>
__device__ __forceinline__ void dft_reg(double2 *v) {
#pragma unroll
    for (int span = R / 2; span >= 1; span >>= 1) {
#pragma unroll
        for (int blk = 0; blk < R; blk += 2 * span) {
#pragma unroll
            for (int i = 0; i < span; ++i) {
                double2 a = v[blk + i], b = v[blk + i + span];
                v[blk + i] = cadd(a, b);
                v[blk + i + span] = mulw16(csub(a, b), i * (8 / span));
            }
        }
    }
    double2 tmp[R];
#pragma unroll
    for (int k = 0; k < R; ++k) tmp[k] = v[brev_c<R>(k)];
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = tmp[k];
}

// omega_n^e from the two-level table: hi[e >> h] * lo[e & (2^h - 1)]
__device__ __forceinline__ double2 tw2(const double2 *__restrict__ hi, const double2 *__restrict__ lo,
                                       uint64_t e, int h) {
    return cmul(__ldg(hi + (e >> h)), __ldg(lo + (e & ((1ull << h) - 1))));
}

// q[r] = omega^(e0 + r*delta) for r < RS, from 1 + log2(RS) table lookups and
// at most log2(RS) products per entry.
template <int RS>
__device__ __forceinline__ void twiddle_run(double2 *q, const PassDesc &d, uint64_t e0, uint64_t delta) {
    q[0] = tw2(d.tw_hi, d.tw_lo, e0 & d.nmask, d.hbits);
    if (RS == 1) return;
    double2 p1 = tw2(d.tw_hi, d.tw_lo, delta & d.nmask, d.hbits);
    q[1] = cmul(q[0], p1);
    if (RS == 2) return;
    double2 p2 = tw2(d.tw_hi, d.tw_lo, (2 * delta) & d.nmask, d.hbits);
    q[2] = cmul(q[0], p2);
    q[3] = cmul(q[1], p2);
    if (RS == 4) return;
    double2 p4 = tw2(d.tw_hi, d.tw_lo, (4 * delta) & d.nmask, d.hbits);
#pragma unroll
    for (int r = 4; r < 8 && r < RS; ++r) q[r] = cmul(q[r - 4], p4);
    if (RS == 8) return;
    double2 p8 = tw2(d.tw_hi, d.tw_lo, (8 * delta) & d.nmask, d.hbits);
#pragma unroll
    for (int r = 8; r < RS; ++r) q[r] = cmul(q[r - 8], p8);
}

// stage twiddles omega_{NsR}^(r*k) = omega_FMAX^(r*e1), e1 = k*FMAX/(Ns*RS): 4 loads + products
template <int RS>
__device__ __forceinline__ void stage_twiddle(double2 *x, const double2 *__restrict__ tf, int e1) {
    if (RS == 1 || e1 == 0) return;
    double2 w1 = __ldg(tf + e1);
    x[1] = cmul(x[1], w1);
    if (RS == 2) return;
    double2 w2 = __ldg(tf + 2 * e1);
    double2 w3 = cmul(w1, w2);
    x[2] = cmul(x[2], w2);
    x[3] = cmul(x[3], w3);
    if (RS == 4) return;
    double2 w4 = __ldg(tf + 4 * e1);
    double2 w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
    x[4] = cmul(x[4], w4);
    x[5] = cmul(x[5], w5);
    x[6] = cmul(x[6], w6);
    x[7] = cmul(x[7], w7);
    if (RS == 8) return;
    double2 w8 = __ldg(tf + 8 * e1);
    x[8] = cmul(x[8], w8);
    x[9] = cmul(x[9], cmul(w1, w8));
    x[10] = cmul(x[10], cmul(w2, w8));
    x[11] = cmul(x[11], cmul(w3, w8));
    x[12] = cmul(x[12], cmul(w4, w8));
    x[13] = cmul(x[13], cmul(w5, w8));
    x[14] = cmul(x[14], cmul(w6, w8));
    x[15] = cmul(x[15], cmul(w7, w8));
}

// shared-memory address of element f of row t: rows padded so T-fastest lane
// groups hit distinct banks; within a row an XOR fold of the 3-bit groups of
// f >> 3 spreads every power-of-two stride over the 8 16-byte bank groups.
template <int F, int T>
__device__ __forceinline__ int smem_idx(int t, int f) {
    constexpr int PAD = T == 1 ? 0 : (T == 2 ? 4 : (T == 4 ? 2 : 1));
    int s = ((f >> 3) ^ (f >> 6) ^ (f >> 9) ^ (f >> 12)) & 7;
    return t * (F + PAD) + (f ^ s);
}

template <int F, int T>
struct PassShape {
    static constexpr int R = F >= 16 ? 16 : F;   // points per thread
    static constexpr int NT = T * F / R;         // threads per CTA
    static constexpr int PAD = T == 1 ? 0 : (T == 2 ? 4 : (T == 4 ? 2 : 1));
    static constexpr size_t SMEM = (F <= 16) ? 0 : (size_t)T * (F + PAD) * sizeof(double2);
    static constexpr int MINB = (T * F <= 2048) ? 4 : ((T * F <= 4096) ? 2 : 1);
};

// Where one tile reads and writes (a persistent kernel retargets these per tile).
//   ld: 0 = ld.global.nc, 1 = ld.global.cg (written earlier in the same launch),
//       2 = ld.global.nc with an L2 evict_first policy (streamed once)
//   st: 0 = st.global, 1 = st.global.cs (streaming), 2 = L2 evict_last policy
struct TileIO {
    const double2 *src;
    double2 *dst;
    int64_t in_shift, out_shift;
};

__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_hint(const double2 *p, unsigned long long pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(double2 *p, double2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}
template <int LD>
__device__ __forceinline__ double2 ld_io(const double2 *p, unsigned long long pol) {
    if constexpr (LD == 1) return __ldcg(p);
    else if constexpr (LD == 2) return ld_hint(p, pol);
    else return __ldg(p);
}
template <int ST>
__device__ __forceinline__ void st_io(double2 *p, double2 v, unsigned long long pol) {
    if constexpr (ST == 1) __stcs(p, v);
    else if constexpr (ST == 2) st_hint(p, v, pol);
    else *p = v;
}

// Input staging layouts of a TMA-loaded tile (SRC != 0):
//   SRC 1 (column tile, box {2T doubles, <=256 points, 1}):   [F][T]
//   SRC 2 (row tile, boxes {<=128 points, T rows} side by side): [F/FB][T][FB], FB = min(F, 128)
template <int F, int T, int SRC>
__device__ __forceinline__ int stage_idx(int t, int f) {
    if constexpr (SRC == 1) {
        return f * T + t;
    } else {
        constexpr int FB = F < 128 ? F : 128;
        return (f / FB) * (T * FB) + t * FB + (f % FB);
    }
}

struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};

// One Stockham stage: Ns = product of the radices already applied.
//   SRC 0: the first stage gathers from global memory; SRC 1/2: from the TMA
//   staging buffer `inbuf`, after which hook() runs (barrier + next prefetch).
template <int F, int T, int NS, bool FIRST, int SRC = 0, class Hook = NoHook, int LD = 0, int ST = 0>
__device__ __forceinline__ void fft_stage(double2 *x, double2 *sm, const PassDesc &d, const TileIO &io,
                                          const double2 *inbuf, const Hook &hook, int64_t in_base,
                                          int64_t k_base, uint64_t al_base, uint64_t be_base) {
    using SH = PassShape<F, T>;
    constexpr int R = SH::R;
    constexpr int NT = SH::NT;
    constexpr int REM = F / NS;
    constexpr int RS = REM >= 16 ? 16 : REM;   // radix of this stage
    constexpr int NB = F / RS;                 // butterflies per transform
    constexpr int M = R / RS;                  // butterflies per thread
    constexpr bool LAST = (NS * RS == F);
    const int tid = threadIdx.x;

    unsigned long long pol = 0;
    if constexpr (FIRST && LD == 2) pol = policy_evict_first();
    if constexpr (LAST && ST == 2) pol = policy_evict_last();
    int tt[M], jj[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        int b = tid + NT * i;
        bool tfast = FIRST ? (SRC == 1 ? true : (SRC == 2 ? false : (bool)d.in_tfast))
                           : (LAST ? d.out_tfast : false);
        if (FIRST && LAST) tfast = d.in_tfast;
        if (tfast) {
            tt[i] = b % T;
            jj[i] = b / T;
        } else {
            tt[i] = b / NB;
            jj[i] = b % NB;
        }
    }
    // ---- gather inputs
#pragma unroll
    for (int i = 0; i < M; ++i) {
#pragma unroll
        for (int r = 0; r < RS; ++r) {
            int f = jj[i] + r * NB;
            double2 val;
            if (FIRST && SRC != 0) {
                val = inbuf[stage_idx<F, T, SRC>(tt[i], f)];
                if (d.conj_in) val.y = -val.y;
            } else if (FIRST) {
                const double2 *p = io.src + (in_base - io.in_shift + (int64_t)tt[i] * d.in_t + (int64_t)f * d.in_f);
                val = ld_io<LD>(p, pol);
                if (d.conj_in) val.y = -val.y;
            } else {
                val = sm[smem_idx<F, T>(tt[i], f)];
            }
            x[i * RS + r] = val;
        }
    }
    if constexpr (FIRST && SRC != 0) hook();
    // ---- twiddle + radix-RS butterflies in registers
#pragma unroll
    for (int i = 0; i < M; ++i) {
        if (NS > 1) stage_twiddle<RS>(x + i * RS, d.tw_f, (jj[i] % NS) * (FMAX / (NS * RS)));
        dft_reg<RS>(x + i * RS);
    }
    if (!LAST) {
        if (!FIRST) __syncthreads();   // every lane has read before anyone overwrites
#pragma unroll
        for (int i = 0; i < M; ++i) {
            int j = jj[i];
            int base = (j / NS) * NS * RS + (j % NS);
#pragma unroll
            for (int r = 0; r < RS; ++r) sm[smem_idx<F, T>(tt[i], base + r * NS)] = x[i * RS + r];
        }
        __syncthreads();
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const int t = tt[i], j = jj[i];
            double2 *v = x + i * RS;
            if (d.twiddle) {
                uint64_t al = al_base + (uint64_t)t * (uint64_t)d.a_t;
                uint64_t be = be_base + (uint64_t)t * (uint64_t)d.b_t;
                double2 q[RS];
                twiddle_run<RS>(q, d, al + be * (uint64_t)j, be * (uint64_t)NB);
#pragma unroll
                for (int r = 0; r < RS; ++r) v[r] = cmul(v[r], q[r]);
            }
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                int64_t k = j + r * NB;
                double2 val = v[r];
                if (d.conj_out) val.y = -val.y;
                int64_t addr;
                if (d.last) {
                    int64_t K = k_base + (int64_t)t * d.K_t + k * d.K_k;
                    addr = d.pack_lp >= 0
                               ? (K & ((1ll << d.pack_lp) - 1)) * d.pack_chunk + (K >> d.pack_lp)
                               : K;
                } else {
                    addr = in_base - io.out_shift + (int64_t)t * d.in_t + k * d.in_f;
                }
                st_io<ST>(io.dst + addr, val, pol);
            }
        }
    }
}

template <int F, int T, int NS, int SRC = 0, class Hook = NoHook, int LD = 0, int ST = 0>
__device__ __forceinline__ void fft_stages(double2 *x, double2 *sm, const PassDesc &d, const TileIO &io,
                                           const double2 *inbuf, const Hook &hook, int64_t in_base,
                                           int64_t k_base, uint64_t al_base, uint64_t be_base) {
    constexpr int REM = F / NS;
    constexpr int RS = REM >= 16 ? 16 : REM;
    fft_stage<F, T, NS, NS == 1, SRC, Hook, LD, ST>(x, sm, d, io, inbuf, hook, in_base, k_base, al_base, be_base);
    if constexpr (NS * RS < F)
        fft_stages<F, T, NS * RS, SRC, Hook, LD, ST>(x, sm, d, io, inbuf, hook, in_base, k_base, al_base,
                                                    be_base);
}

// one tile of T transforms; tile id -> (u, v, w) as documented in PassDesc
template <int F, int T, int SRC = 0, class Hook = NoHook, int LD = 0, int ST = 0>
__device__ __forceinline__ void tile_fft(double2 *sm, const PassDesc &d, const TileIO &io, int64_t b,
                                         const double2 *inbuf = nullptr, const Hook &hook = Hook()) {
    const int64_t u = b % d.U;
    b /= d.U;
    const int64_t v = b % d.V;
    const int64_t w = b / d.V;
    const int64_t in_base = u * d.in_u + v * d.in_v + w * d.in_w;
    const int64_t k_base = u * d.K_u + v * d.K_v + w * d.K_w;
    const uint64_t al_base = (uint64_t)d.a_c + (uint64_t)u * d.a_u + (uint64_t)v * d.a_v + (uint64_t)w * d.a_w;
    const uint64_t be_base = (uint64_t)d.b_c + (uint64_t)u * d.b_u + (uint64_t)v * d.b_v + (uint64_t)w * d.b_w;
    double2 x[PassShape<F, T>::R];
    fft_stages<F, T, 1, SRC, Hook, LD, ST>(x, sm, d, io, inbuf, hook, in_base, k_base, al_base, be_base);
}

template <int F, int T>
__global__ void __launch_bounds__(PassShape<F, T>::NT, PassShape<F, T>::MINB)
    fft_pass_kernel(const PassDesc d) {
    extern __shared__ double2 sm[];
    TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    tile_fft<F, T>(sm, d, io, blockIdx.x);
}

template <int F, int T>
cudaError_t launch_one(const PassDesc &d, int64_t tiles, cudaStream_t s) {
    using SH = PassShape<F, T>;
    fft_pass_kernel<F, T><<<(unsigned)tiles, SH::NT, SH::SMEM, s>>>(d);
    return cudaGetLastError();
}

template <int F, int T>
cudaError_t prepare_one() {
    using SH = PassShape<F, T>;
    if (SH::SMEM > 48 * 1024)
        return cudaFuncSetAttribute(fft_pass_kernel<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SH::SMEM);
    return cudaSuccess;
}

}  // namespace moa

namespace moa {

// ---------------------------------------------------------------------------
// Persistent TMA pass: one CTA per SM slot walks tiles blockIdx.x, +gridDim.x, ...
// The tile is copied global -> shared by cp.async.bulk.tensor (one elected
// thread, mbarrier completion); as soon as the first butterfly stage has read
// it into registers the copy of the CTA's next tile is issued, so HBM reads
// overlap the FP64 butterflies, the shared-memory exchanges and the stores.
template <int F, int T, int SRC>
struct TmaShape {
    static constexpr int FB = SRC == 1 ? (F < 256 ? F : 256) : (F < 128 ? F : 128);   // points per box
    static constexpr int NBOX = F / FB;
    static constexpr unsigned BOX_BYTES = (unsigned)(FB * T * 16);
    static constexpr size_t IN_BYTES = (size_t)T * F * 16;
    static constexpr size_t SMEM = 128 + IN_BYTES + PassShape<F, T>::SMEM + 16;
};

template <int F, int T, int SRC>
__device__ __forceinline__ void tma_issue_tile(const CUtensorMap *map, uint64_t *bar, double2 *inbuf,
                                               const PassDesc &d, int64_t tile) {
    using TS = TmaShape<F, T, SRC>;
    int64_t b = tile;
    const int u = (int)(b % d.U);
    b /= d.U;
    const int v = (int)(b % d.V);
    const int w = (int)(b / d.V);
    mbar_expect_tx(bar, TS::BOX_BYTES * TS::NBOX);
#pragma unroll
    for (int k = 0; k < TS::NBOX; ++k) {
        if constexpr (SRC == 1)   // column tile: dims {2B doubles, F, A}
            tma_load_3d(inbuf + k * TS::FB * T, map, bar, 2 * T * u, k * TS::FB, v);
        else                      // row tile: dims {2F doubles, rows, V, W}
            tma_load_4d(inbuf + k * TS::FB * T, map, bar, 2 * TS::FB * k, T * u, v, w);
    }
}

template <int F, int T, int SRC>
__global__ void __launch_bounds__(PassShape<F, T>::NT, 1)
    fft_pass_tma_kernel(const PassDesc d, const __grid_constant__ CUtensorMap tmap, int64_t tiles) {
    extern __shared__ unsigned char smraw[];
    double2 *inbuf = reinterpret_cast<double2 *>((reinterpret_cast<uintptr_t>(smraw) + 127) & ~uintptr_t(127));
    double2 *work = inbuf + T * F;
    uint64_t *bar = reinterpret_cast<uint64_t *>(work + (PassShape<F, T>::SMEM / sizeof(double2)));
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    int64_t tile = blockIdx.x;
    if (tid == 0 && tile < tiles) tma_issue_tile<F, T, SRC>(&tmap, bar, inbuf, d, tile);
    const TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    unsigned phase = 0;
    for (; tile < tiles; tile += gridDim.x) {
        mbar_wait(bar, phase);
        phase ^= 1;
        const int64_t next = tile + gridDim.x;
        auto hook = [&]() {
            __syncthreads();   // every lane has its inputs in registers: the staging buffer is free
            if (tid == 0 && next < tiles) {
                fence_proxy_async();
                tma_issue_tile<F, T, SRC>(&tmap, bar, inbuf, d, next);
            }
        };
        tile_fft<F, T, SRC>(work, d, io, tile, inbuf, hook);
    }
}

template <int F, int T, int SRC>
cudaError_t launch_one_tma(const PassDesc &d, const CUtensorMap &map, int64_t tiles, int grid, cudaStream_t s) {
    using TS = TmaShape<F, T, SRC>;
    fft_pass_tma_kernel<F, T, SRC><<<grid, PassShape<F, T>::NT, TS::SMEM, s>>>(d, map, tiles);
    return cudaGetLastError();
}

template <int F, int T, int SRC>
int grid_one_tma() {
    using TS = TmaShape<F, T, SRC>;
    if (TS::SMEM > 48 * 1024 &&
        cudaFuncSetAttribute(fft_pass_tma_kernel<F, T, SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)TS::SMEM) != cudaSuccess)
        return 0;
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft_pass_tma_kernel<F, T, SRC>,
                                                      PassShape<F, T>::NT, TS::SMEM) != cudaSuccess)
        return 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}

}  // namespace moa
