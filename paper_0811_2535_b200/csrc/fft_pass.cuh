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
#include <stdlib.h>

// points per thread (the largest in-register radix).  Measured: 8 points per thread
// (1024 threads/SM at <= 64 registers) is 20-35 % slower than 16 on B200.
#define MOA_RMAX 16

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

// p + off elements with a 32-bit element offset: one IMAD.WIDE.U32 per address
// (the byte offset itself may exceed 32 bits)
template <class Tp>
__device__ __forceinline__ Tp *elem_off(Tp *p, uint32_t off) {
    return reinterpret_cast<Tp *>(reinterpret_cast<uintptr_t>(p) + (uint64_t)off * 16u);
}
// p + c * stride elements, c a compile-time constant
template <class Tp>
__device__ __forceinline__ Tp *elem_off_c(Tp *p, uint32_t c, uint32_t stride) {
    return reinterpret_cast<Tp *>(reinterpret_cast<uintptr_t>(p) + (uint64_t)(16u * c) * (uint64_t)stride);
}


// stage twiddles omega_{Ns*RS}^(r*k) = omega_FMAX^(r*e1), e1 = k*FMAX/(Ns*RS): 4 table
// loads (r = 1, 2, 4, 8) and products for the rest.  (One table load per point was
// measured slower: more loads on the latency-critical path between the stages.)
// stage_twiddle with the pass twiddle's butterfly-constant factor a = omega^(al+be*j)
// folded in (last stage of a twiddled pass): x[s] *= a * omega_F^(j*s).  DFT linearity
// moves a from the 16 outputs to the 16 inputs, where it rides on the stage twiddles'
// power chain (c_s = c_lo * w_hi): 16 + 4 products instead of 15 + 16.
template <int RS>
__device__ __forceinline__ void stage_twiddle_scaled(double2 *x, const double2 *__restrict__ tf, int e1, double2 a) {
    x[0] = cmul(x[0], a);
    if (RS == 1) return;
    double2 w1 = __ldg(tf + e1);
    double2 w2 = RS > 2 ? __ldg(tf + 2 * e1) : w1;
    double2 w4 = RS > 4 ? __ldg(tf + 4 * e1) : w1;
    double2 w8 = RS > 8 ? __ldg(tf + 8 * e1) : w1;
    double2 c1 = cmul(a, w1);
    x[1] = cmul(x[1], c1);
    if (RS == 2) return;
    double2 c2 = cmul(a, w2), c3 = cmul(c1, w2);
    x[2] = cmul(x[2], c2);
    x[3] = cmul(x[3], c3);
    if (RS == 4) return;
    double2 c4 = cmul(a, w4), c5 = cmul(c1, w4), c6 = cmul(c2, w4), c7 = cmul(c3, w4);
    x[4] = cmul(x[4], c4);
    x[5] = cmul(x[5], c5);
    x[6] = cmul(x[6], c6);
    x[7] = cmul(x[7], c7);
    if (RS == 8) return;
    x[8] = cmul(x[8], cmul(a, w8));
    x[9] = cmul(x[9], cmul(c1, w8));
    x[10] = cmul(x[10], cmul(c2, w8));
    x[11] = cmul(x[11], cmul(c3, w8));
    x[12] = cmul(x[12], cmul(c4, w8));
    x[13] = cmul(x[13], cmul(c5, w8));
    x[14] = cmul(x[14], cmul(c6, w8));
    x[15] = cmul(x[15], cmul(c7, w8));
}

template <int RS>
__device__ __forceinline__ void stage_twiddle(double2 *x, const double2 *__restrict__ tf, int e1) {
    if (RS == 1) return;   // (no e1 == 0 shortcut: a divergent exit costs more register moves than it saves)
    double2 w1 = __ldg(tf + e1);
    double2 w2 = RS > 2 ? __ldg(tf + 2 * e1) : w1;
    double2 w4 = RS > 4 ? __ldg(tf + 4 * e1) : w1;
    double2 w8 = RS > 8 ? __ldg(tf + 8 * e1) : w1;
    x[1] = cmul(x[1], w1);
    if (RS == 2) return;
    double2 w3 = cmul(w1, w2);
    x[2] = cmul(x[2], w2);
    x[3] = cmul(x[3], w3);
    if (RS == 4) return;
    double2 w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
    x[4] = cmul(x[4], w4);
    x[5] = cmul(x[5], w5);
    x[6] = cmul(x[6], w6);
    x[7] = cmul(x[7], w7);
    if (RS == 8) return;
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
    int s = ((f >> 3) ^ (f >> 6) ^ (f >> 9) ^ (f >> 12)) & 7;   // == swz(f)
    return t * (F + PAD) + (f ^ s);
}

// Radix of the Stockham stage that starts once NS points have been combined.
// F a power of 16 (or < 32): radix 16 throughout.  Otherwise the remainder FIRST, then
// radix 16, so the last stage is radix 16 and the per-tile pass-twiddle table holds F/16
// entries per transform (measured faster than remainder-last at every F).
__host__ __device__ constexpr int first_radix(int F) {
    int r = F;
    while (r > MOA_RMAX) r /= MOA_RMAX;
    return r;
}
#ifndef MOA_RF_MIN
#define MOA_RF_MIN 32
#endif
__host__ __device__ constexpr bool remainder_first(int F) { return F >= MOA_RF_MIN && first_radix(F) != MOA_RMAX; }
__host__ __device__ constexpr int stage_radix(int F, int NS) {
    if (remainder_first(F)) return NS == 1 ? first_radix(F) : MOA_RMAX;
    return F / NS >= MOA_RMAX ? MOA_RMAX : F / NS;
}
// radix of the last stage
__host__ __device__ constexpr int lrs(int F) {
    if (remainder_first(F)) return MOA_RMAX;
    int ns = 1;
    while (F / ns > MOA_RMAX) ns *= MOA_RMAX;
    return F / ns;
}

// NS of the stage that wrote the exchange read by the stage starting at NS (0: none)
__host__ __device__ constexpr int writer_ns(int F, int NS) {
    int ns = 1;
    if (NS <= 1) return 0;
    while (ns * stage_radix(F, ns) < NS) ns *= stage_radix(F, ns);
    return ns;
}
// Extra bank-group XOR for an exchange written by a radix-16 stage with NS = 2 or 4 (the
// stage after a radix-2/4 remainder stage, F = 512, 1024, 8192): its quarter-warp lanes
// differ in point bits {0, 5, 6} (NS = 2) or {0, 1, 6} (NS = 4), which swz() maps onto 4
// bank groups; bit 6 goes to the bank bit swz leaves constant (tools/bank_sim.py:
// F = 1024 stores 2.0 -> 1.0 wavefronts per ideal in that stage, no other pattern changes).
template <int NSW>
__device__ __forceinline__ int xmask(int f) {
    if constexpr (NSW == 4) return ((f >> 6) & 1) << 2;
    if constexpr (NSW == 2) return ((f >> 6) & 1) << 1;
    return 0;
}

template <int F, int T>
struct PassShape {
    static constexpr int R = F >= MOA_RMAX ? MOA_RMAX : F;   // points per thread
    static constexpr int NT = T * F / R;         // threads per CTA
    static constexpr int PAD = T == 1 ? 0 : (T == 2 ? 4 : (T == 4 ? 2 : 1));
    // last-stage geometry (for the per-tile twiddle tables)
    static constexpr int LRS = lrs(F);
    static constexpr int LNB = F / LRS;
    static constexpr size_t XCH = (F <= 16) ? 0 : (size_t)T * (F + PAD) * sizeof(double2);   // exchange buffer
    static constexpr size_t TWA = (size_t)T * (LNB + 1) * sizeof(double2);   // A[t][j] = w^(al_t + be_t j)
    static constexpr size_t TWB = (size_t)T * (LRS + 1) * sizeof(double2);   // B[t][r] = w^(be_t NB r)
    static constexpr size_t SMEM = XCH + TWA + TWB;
    // resident threads per SM: 512 at 16 points per thread (<= 128 registers each),
    // 1024 at 8 points per thread (<= 64 registers)
    static constexpr int TGT = 512 * 16 / MOA_RMAX;
    static constexpr int MINB = TGT / NT < 1 ? 1 : (TGT / NT > 16 ? 16 : TGT / NT);
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
    else   // explicit st.global (a peer pointer must not become a generic store)
        asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
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

// ST = 4: the last stage's output tensor map (a no-op hook otherwise)
struct OMapHook {
    const CUtensorMap *m;
    __device__ __forceinline__ void operator()() const {}
};

struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};

// XOR-fold swizzle of a row-local point index (see smem_idx)
__host__ __device__ constexpr int swz(int f) { return ((f >> 3) ^ (f >> 6) ^ (f >> 9) ^ (f >> 12)) & 7; }


// Per-tile values shared by the stages of one tile.
struct TileCtx {
    const double2 *in;   // src + tile input base  (element (t, f) at in[t*in_t + f*in_f])
    double2 *out;        // dst + tile output base (element (t, k) at out[t*out_t + k*out_k])
    int64_t k_base;      // general pack path only
    uint32_t al, be;     // twiddle exponent: omega_n^(al + a_t*t + (be + b_t*t)*k)
    const double2 *twa;  // shared A[t][j], pitch LNB+1
    const double2 *twb;  // shared B[t][r], pitch LRS+1
};

// omega_n^e = exp(-2 pi i e / n) evaluated directly: sincospi of the exact
// rational -2e/n (no table, no memory latency; CUDA's sincospi is within 1 ulp)
__device__ __forceinline__ double2 root_pi(uint32_t e, int t) {
    double s, c;
    sincospi(-ldexp((double)e, 1 - t), &s, &c);
    return make_double2(c, s);
}

// Build the tile's twiddle tables: omega^(al_t + be_t*(j + r*NB)) = A[t][j] * B[t][r],
// each entry by sincospi of the exact rational exponent (FP64 work, no loads: a lookup in
// the plan's two-level omega_n table was measured slower, its loads sit on the tile's
// critical path); the stages' barriers publish the tables.
template <int F, int T>
__device__ __forceinline__ void build_twiddle_tables(const PassDesc &d, double2 *twa, double2 *twb, uint32_t al,
                                                     uint32_t be) {
    using SH = PassShape<F, T>;
    constexpr int NB = SH::LNB, RS = SH::LRS;
    const uint32_t nm = (uint32_t)d.nmask;
    for (int i = threadIdx.x; i < T * (NB + RS); i += SH::NT) {
        if (i < T * NB) {
            const int t = i / NB, j = i % NB;
            const uint32_t a = al + (uint32_t)t * (uint32_t)d.a_t, b = be + (uint32_t)t * (uint32_t)d.b_t;
            twa[t * (NB + 1) + j] = root_pi((a + b * (uint32_t)j) & nm, d.tbits);
        } else {
            const int k = i - T * NB, t = k / RS, r = k % RS;
            const uint32_t b = be + (uint32_t)t * (uint32_t)d.b_t;
            twb[t * (RS + 1) + r] = root_pi((b * (uint32_t)(NB * r)) & nm, d.tbits);
        }
    }
}

// The first stage's gather of `tile` into registers (lane mapping of the SRC 0 stage).
template <int F, int T>
__device__ __forceinline__ void rdb_load_tile(double2 *x, const PassDesc &d, const TileIO &io, int64_t b) {
    using SH = PassShape<F, T>;
    constexpr int RS = stage_radix(F, 1), NB = F / RS, M = SH::R / RS, NT = SH::NT;
    const int64_t u = b & (d.U - 1);
    const int64_t v = (b >> d.lU) & (d.V - 1);
    const int64_t w = b >> (d.lU + d.lV);
    const double2 *in = io.src + (u * d.in_u + v * d.in_v + w * d.in_w - io.in_shift);
    const uint32_t sf = (uint32_t)NB * (uint32_t)d.in_f;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const int bb = threadIdx.x + NT * i;
        const bool tfast = T > 1 && d.in_tfast;
        const int t = tfast ? bb % T : bb / NB, j = tfast ? bb / T : bb % NB;
        const double2 *p = elem_off(in, (uint32_t)t * (uint32_t)d.in_t + (uint32_t)j * (uint32_t)d.in_f);
#pragma unroll
        for (int r = 0; r < RS; ++r) x[i * RS + r] = __ldg(elem_off_c(p, r, sf));
    }
}

// One Stockham stage: Ns = product of the radices already applied.
//   SRC 0: the first stage gathers from global memory; SRC 1/2: from the TMA
//   staging buffer `inbuf`, after which hook() runs (barrier + next prefetch).
// Address arithmetic is split into a per-butterfly part and compile-time
// per-point constants: global addresses are base + r*(NB*stride); shared
// addresses use phys(j + r*NB) = (j ^ swz(j) ^ swz(r*NB)) + r*NB (the XOR fold is
// linear over the disjoint bit fields of j and r*NB).
// TW: 0 = the pass has no twiddle, 1 = it has one (both compile-time: no uniform branch
// whose two register assignments the compiler must reconcile), 2 = d.twiddle at run time
template <int F, int T, int NS, bool FIRST, int SRC = 0, class Hook = NoHook, int LD = 0, int ST = 0, int TW = 2>
__device__ __forceinline__ void fft_stage(double2 *x, double2 *sm, const PassDesc &d, const TileCtx &c,
                                          const double2 *inbuf, const Hook &hook) {
    using SH = PassShape<F, T>;
    constexpr int R = SH::R;
    constexpr int NT = SH::NT;
    constexpr int REM = F / NS;
    constexpr int RS = stage_radix(F, NS);   // radix of this stage
    constexpr int NB = F / RS;                 // butterflies per transform
    constexpr int M = R / RS;                  // butterflies per thread
    constexpr bool LAST = (NS * RS == F);
    constexpr int ROW = F + SH::PAD;           // shared row pitch
    const int tid = threadIdx.x;
    // staging layout of a TMA-loaded tile: SRC 4/5 (single buffer, prefetch after the
    // last stage's reads) stage like SRC 1/2 (column / row tiles)
    constexpr int SL = SRC == 4 ? 1 : (SRC == 5 ? 2 : SRC);

    unsigned long long pol = 0;
    if constexpr (FIRST && LD == 2) pol = policy_evict_first();
    if constexpr (LAST && ST == 2) pol = policy_evict_last();
    int tt[M], jj[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        int b = tid + NT * i;
        bool tfast = FIRST ? (SL == 1 ? true : (SL == 2 ? false : (bool)d.in_tfast))
                           : (LAST ? (bool)d.out_tfast : false);
        if (FIRST && LAST) tfast = SL == 1 ? true : (SL == 2 ? false : (bool)d.in_tfast);
        if (T == 1) tfast = false;
        if (tfast) {
            tt[i] = b % T;
            jj[i] = b / T;
        } else {
            tt[i] = b / NB;
            jj[i] = b % NB;
        }
    }
    // ---- gather inputs (the first stage then builds the tile's twiddle tables while
    //      its loads are in flight)
    if constexpr (FIRST && SRC == 0) {
        // element offsets inside the tile's span fit 32 bits (span < n <= 2^32)
        const uint32_t sf = (uint32_t)NB * (uint32_t)d.in_f;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const double2 *p = elem_off(c.in, (uint32_t)tt[i] * (uint32_t)d.in_t + (uint32_t)jj[i] * (uint32_t)d.in_f);
#pragma unroll
            for (int r = 0; r < RS; ++r) x[i * RS + r] = ld_io<LD>(elem_off_c(p, r, sf), pol);
        }
        if (d.conj_in) {
#pragma unroll
            for (int k = 0; k < R; ++k) x[k].y = -x[k].y;
        }
        if (TW == 1 || (TW == 2 && d.twiddle))
            build_twiddle_tables<F, T>(d, const_cast<double2 *>(c.twa), const_cast<double2 *>(c.twb), c.al, c.be);
        if constexpr (LAST) __syncthreads();   // single-stage transform: publish the tables
    } else if constexpr (FIRST && SRC == 6) {
        // register double buffering (fft_pass_rdb_kernel): this tile's points were loaded
        // into the hook's registers during the previous tile; take them and start the
        // loads of the CTA's next tile into the same registers at once
        hook.take(x);
        hook.prefetch();
        if (d.conj_in) {
#pragma unroll
            for (int k = 0; k < R; ++k) x[k].y = -x[k].y;
        }
        if (TW == 1 || (TW == 2 && d.twiddle))
            build_twiddle_tables<F, T>(d, const_cast<double2 *>(c.twa), const_cast<double2 *>(c.twb), c.al, c.be);
    } else if constexpr (FIRST && SRC == 3) {
        // prefetched by this same thread (cp.async, fft_pass_pf_kernel) into the
        // exchange layout: its own copies are visible after cp.async.wait_all
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int r = 0; r < RS; ++r) x[i * RS + r] = sm[smem_idx<F, T>(tt[i], jj[i] + r * NB)];
        if (d.conj_in) {
#pragma unroll
            for (int k = 0; k < R; ++k) x[k].y = -x[k].y;
        }
        if (TW == 1 || (TW == 2 && d.twiddle))
            build_twiddle_tables<F, T>(d, const_cast<double2 *>(c.twa), const_cast<double2 *>(c.twb), c.al, c.be);
    } else if constexpr (FIRST) {
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int r = 0; r < RS; ++r) x[i * RS + r] = inbuf[stage_idx<F, T, SL>(tt[i], jj[i] + r * NB)];
        if (d.conj_in) {
#pragma unroll
            for (int k = 0; k < R; ++k) x[k].y = -x[k].y;
        }
        if (TW == 1 || (TW == 2 && d.twiddle))
            build_twiddle_tables<F, T>(d, const_cast<double2 *>(c.twa), const_cast<double2 *>(c.twb), c.al, c.be);
        if constexpr (SRC <= 2) hook();
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const int j = jj[i];
            if constexpr (NB >= 8) {
                constexpr int NSW = writer_ns(F, NS);
                const int rowoff = tt[i] * ROW, pj = j ^ swz(j);
#pragma unroll
                for (int r = 0; r < RS; ++r)
                    x[i * RS + r] = sm[rowoff + ((pj ^ swz(r * NB) ^ xmask<NSW>(j + r * NB)) + r * NB)];
            } else {
#pragma unroll
                for (int r = 0; r < RS; ++r) x[i * RS + r] = sm[smem_idx<F, T>(tt[i], j + r * NB)];
            }
        }
        // the exchange buffer is free once every lane has read it: the prefetching
        // kernel starts the next tile's copy into it here (hook = barrier + cp.async)
        if constexpr (LAST && SRC >= 3) hook();
    }
    // ---- twiddle + radix-RS butterflies in registers (FOLD: the last stage of a
    //      twiddled pass takes the pass twiddle's factor A[t][j] on its inputs)
    constexpr bool FOLD = LAST && NS > 1 && TW == 1;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        if constexpr (FOLD)
            stage_twiddle_scaled<RS>(x + i * RS, d.tw_f, (jj[i] % NS) * (FMAX / (NS * RS)),
                                     c.twa[tt[i] * (NB + 1) + jj[i]]);
        else if (NS > 1)
            stage_twiddle<RS>(x + i * RS, d.tw_f, (jj[i] % NS) * (FMAX / (NS * RS)));
        dft_reg<RS>(x + i * RS);
    }
    if constexpr (!LAST) {
        if (!FIRST || SRC >= 3) __syncthreads();   // every lane has read before anyone overwrites
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const int j = jj[i];
            const int base = (j / NS) * NS * RS + (j % NS);
            if constexpr (NS >= 8) {
                const int rowoff = tt[i] * ROW, pb = base ^ swz(base);
#pragma unroll
                for (int r = 0; r < RS; ++r) sm[rowoff + ((pb ^ swz(r * NS)) + r * NS)] = x[i * RS + r];
            } else if constexpr (NS == 1 && RS >= 8) {
                const int pb = tt[i] * ROW + base;
                const int sb = swz(base);
#pragma unroll
                for (int r = 0; r < RS; ++r) sm[pb + (r ^ sb ^ swz(r))] = x[i * RS + r];
            } else if constexpr (NS == 2 || NS == 4) {
                const int rowoff = tt[i] * ROW;
#pragma unroll
                for (int r = 0; r < RS; ++r) {
                    const int f = base + r * NS;
                    sm[rowoff + (f ^ swz(f) ^ xmask<NS>(f))] = x[i * RS + r];
                }
            } else {
#pragma unroll
                for (int r = 0; r < RS; ++r) sm[smem_idx<F, T>(tt[i], base + r * NS)] = x[i * RS + r];
            }
        }
        __syncthreads();
    } else {
        const uint32_t so = (uint32_t)NB * (uint32_t)d.out_k;
        if constexpr (ST == 4) __syncthreads();   // every lane has read the exchange buffer
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const int t = tt[i], j = jj[i];
            double2 *v = x + i * RS;
            if constexpr (FOLD) {   // output r: times B[t][r] (B[t][0] = 1)
#pragma unroll
                for (int r = 1; r < RS; ++r) v[r] = cmul(v[r], c.twb[t * (RS + 1) + r]);
            } else if (TW == 1 || (TW == 2 && d.twiddle)) {
                const double2 a = c.twa[t * (NB + 1) + j];
                v[0] = cmul(v[0], a);
#pragma unroll
                for (int r = 1; r < RS; ++r) v[r] = cmul(v[r], cmul(a, c.twb[t * (RS + 1) + r]));
            }
            if (d.conj_out) {
#pragma unroll
                for (int r = 0; r < RS; ++r) v[r].y = -v[r].y;
            }
            if constexpr (ST == 4) {   // stage [k][t] for the bulk-tensor store
#pragma unroll
                for (int r = 0; r < RS; ++r) sm[(j + r * NB) * T + t] = v[r];
                continue;
            }
            if (d.pack_lp >= 0) {   // general pack (single-level local transform, p > 1)
#pragma unroll
                for (int r = 0; r < RS; ++r) {
                    const int64_t K = c.k_base + (int64_t)t * d.K_t + (int64_t)(j + r * NB) * d.K_k;
                    const int64_t dst = K & ((1ll << d.pack_lp) - 1);
                    double2 *a = d.peer[0] ? d.peer[dst] + (d.peer_off + (K >> d.pack_lp))
                                           : c.out + (dst * d.pack_chunk + (K >> d.pack_lp));
                    st_io<ST>(a, v[r], pol);
                }
            } else {
                double2 *po = elem_off(c.out, (uint32_t)t * (uint32_t)d.out_t + (uint32_t)j * (uint32_t)d.out_k);
#pragma unroll
                for (int r = 0; r < RS; ++r) st_io<ST>(elem_off_c(po, r, so), v[r], pol);
            }
        }
        if constexpr (ST == 4) {
            // boxes of KB k-rows x T points: output inner index c.k_base + t (runs of T),
            // outer index k (stride K_k); one thread hands them to the TMA engine
            constexpr int KB = F < 256 ? F : 256;
            fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
#pragma unroll 1
                for (int kb = 0; kb < F / KB; ++kb)
                    tma_store_2d(hook.m, sm + kb * KB * T, 2 * (int)c.k_base, kb * KB);
                tma_store_drain();
            }
        }
    }
}

template <int F, int T, int NS, int SRC = 0, class Hook = NoHook, int LD = 0, int ST = 0, int TW = 2>
__device__ __forceinline__ void fft_stages(double2 *x, double2 *sm, const PassDesc &d, const TileCtx &c,
                                           const double2 *inbuf, const Hook &hook) {
    constexpr int RS = stage_radix(F, NS);
    fft_stage<F, T, NS, NS == 1, SRC, Hook, LD, ST, TW>(x, sm, d, c, inbuf, hook);
    if constexpr (NS * RS < F) fft_stages<F, T, NS * RS, SRC, Hook, LD, ST, TW>(x, sm, d, c, inbuf, hook);
}

// one tile of T transforms; tile id -> (u, v, w) as documented in PassDesc
template <int F, int T, int SRC = 0, class Hook = NoHook, int LD = 0, int ST = 0, int TW = 2>
__device__ __forceinline__ void tile_fft(double2 *sm, double2 *tw, const PassDesc &d, const TileIO &io, int64_t b,
                                         const double2 *inbuf = nullptr, const Hook &hook = Hook()) {
    // batch index above the per-transform tile bits
    int64_t boff = 0;
    if (d.bstride) {
        boff = (b >> d.ltiles) * d.bstride;
        b &= ((int64_t)1 << d.ltiles) - 1;
    }
    // U and V are powers of two: decode with shifts and masks
    const int64_t u = b & (d.U - 1);
    const int64_t v = (b >> d.lU) & (d.V - 1);
    const int64_t w = b >> (d.lU + d.lV);
    TileCtx c;
    c.in = io.src + (boff + u * d.in_u + v * d.in_v + w * d.in_w - io.in_shift);
    // fused exchange: tile row v is destination rank v (every row of the tile goes there)
    c.out = d.peer[0] ? d.peer[v] + (d.peer_off + u * d.out_u + w * d.out_w)
                      : io.dst + (boff + u * d.out_u + v * d.out_v + w * d.out_w - io.out_shift);
    c.k_base = u * d.K_u + v * d.K_v + w * d.K_w;
    c.al = (uint32_t)d.a_c + (uint32_t)u * (uint32_t)d.a_u + (uint32_t)v * (uint32_t)d.a_v + (uint32_t)w * (uint32_t)d.a_w;
    c.be = (uint32_t)d.b_c + (uint32_t)u * (uint32_t)d.b_u + (uint32_t)v * (uint32_t)d.b_v + (uint32_t)w * (uint32_t)d.b_w;
    using SH = PassShape<F, T>;
    double2 *twa = tw;
    double2 *twb = twa + SH::TWA / sizeof(double2);
    c.twa = twa;
    c.twb = twb;
    double2 x[PassShape<F, T>::R];
    fft_stages<F, T, 1, SRC, Hook, LD, ST, TW>(x, sm, d, c, inbuf, hook);
}

template <int F, int T, int TW>
__global__ void __launch_bounds__(PassShape<F, T>::NT, PassShape<F, T>::MINB)
    fft_pass_kernel(const PassDesc d) {
    extern __shared__ double2 sm[];
    if (d.pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    tile_fft<F, T, 0, NoHook, 0, 0, TW>(sm, reinterpret_cast<double2 *>(reinterpret_cast<char *>(sm) + PassShape<F, T>::XCH), d, io,
                   blockIdx.x);
}

// Row pass whose transposed store goes through shared memory and the TMA engine
// (cp.async.bulk.tensor stores of KB k-rows x T points) instead of per-lane st.global.
template <int F, int T, int TW>
__global__ void __launch_bounds__(PassShape<F, T>::NT, PassShape<F, T>::MINB)
    fft_pass_tmast_kernel(const PassDesc d, const __grid_constant__ CUtensorMap omap) {
    extern __shared__ double2 sm[];
    if (d.pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    tile_fft<F, T, 0, OMapHook, 0, 4, TW>(sm, reinterpret_cast<double2 *>(reinterpret_cast<char *>(sm) + PassShape<F, T>::XCH),
                                          d, io, blockIdx.x, nullptr, OMapHook{&omap});
}

template <int F, int T>
cudaError_t launch_tmast(const PassDesc &d, const CUtensorMap &omap, int64_t tiles, cudaStream_t s) {
    using SH = PassShape<F, T>;
    auto kernel = d.twiddle ? fft_pass_tmast_kernel<F, T, 1> : fft_pass_tmast_kernel<F, T, 0>;
    // (the shared-memory limit is raised per device by prepare_one, plan.cu)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tiles);
    cfg.blockDim = dim3(SH::NT);
    cfg.dynamicSmemBytes = SH::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = d.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, d, omap);
}

#ifdef MOA_VARIANTS
// ---------------------------------------------------------------------------
// Persistent pass with the next tile prefetched into the exchange buffer.
// The exchange buffer is idle from the moment the last stage has read it until
// the next tile's first stage: each thread starts cp.async copies of its share of
// the next tile there (global -> shared, no registers held), so the HBM latency
// of tile i+1 overlaps the last butterflies, the twiddles and the stores of tile
// i.  Same shared memory and registers as fft_pass_kernel (4 CTAs per SM at
// F*T = 2048), one CTA per resident slot.
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// this thread's share of `tile`, in the first stage's lane mapping and the exchange layout
template <int F, int T>
__device__ __forceinline__ void prefetch_tile(double2 *sm, const PassDesc &d, const TileIO &io, int64_t b) {
    using SH = PassShape<F, T>;
    constexpr int RS = stage_radix(F, 1), NB = F / RS, M = SH::R / RS, NT = SH::NT;
    const int64_t u = b & (d.U - 1);
    const int64_t v = (b >> d.lU) & (d.V - 1);
    const int64_t w = b >> (d.lU + d.lV);
    const double2 *in = io.src + (u * d.in_u + v * d.in_v + w * d.in_w - io.in_shift);
    const uint32_t sf = (uint32_t)NB * (uint32_t)d.in_f;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const int bb = threadIdx.x + NT * i;
        const bool tfast = T > 1 && d.in_tfast;
        const int t = tfast ? bb % T : bb / NB, j = tfast ? bb / T : bb % NB;
        const double2 *p = elem_off(in, (uint32_t)t * (uint32_t)d.in_t + (uint32_t)j * (uint32_t)d.in_f);
#pragma unroll
        for (int r = 0; r < RS; ++r) cp_async16(sm + smem_idx<F, T>(t, j + r * NB), elem_off_c(p, r, sf));
    }
}

template <int F, int T>
struct PrefetchHook {
    double2 *sm;
    const PassDesc *d;
    const TileIO *io;
    int64_t next, tiles;
    __device__ __forceinline__ void operator()() const {
        __syncthreads();   // every lane has read the exchange buffer
        if (next < tiles) prefetch_tile<F, T>(sm, *d, *io, next);
        cp_async_commit();
    }
};

template <int F, int T>
__global__ void __launch_bounds__(PassShape<F, T>::NT, PassShape<F, T>::MINB)
    fft_pass_pf_kernel(const PassDesc d, int64_t tiles) {
    extern __shared__ double2 sm[];
    double2 *tw = reinterpret_cast<double2 *>(reinterpret_cast<char *>(sm) + PassShape<F, T>::XCH);
    const TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    int64_t tile = blockIdx.x;
    if (tile >= tiles) return;
    prefetch_tile<F, T>(sm, d, io, tile);
    cp_async_commit();
    for (; tile < tiles; tile += gridDim.x) {
        cp_async_wait_all();
        __syncthreads();   // the previous tile's epilogue is done with the twiddle tables
        const PrefetchHook<F, T> hk{sm, &d, &io, tile + (int64_t)gridDim.x, tiles};
        tile_fft<F, T, 3, PrefetchHook<F, T>>(sm, tw, d, io, tile, nullptr, hk);
    }
}

// ---------------------------------------------------------------------------
// Register double buffering: a persistent CTA holds the NEXT tile's points in a second
// register set; the loads for tile i+1 are issued as soon as tile i's points have been
// taken out of it, so they overlap all of tile i's butterflies, exchange and stores.
// 3 CTAs/SM (<= 170 registers: two 16-point sets per thread).
template <int F, int T>
struct RdbHook {
    double2 *nx;   // PassShape<F,T>::R registers (fully unrolled, never indexed dynamically)
    const PassDesc *d;
    const TileIO *io;
    int64_t next, tiles;
    __device__ __forceinline__ void take(double2 *x) const {
#pragma unroll
        for (int k = 0; k < PassShape<F, T>::R; ++k) x[k] = nx[k];
    }
    __device__ __forceinline__ void prefetch() const {
        if (next < tiles) rdb_load_tile<F, T>(nx, *d, *io, next);
    }
    __device__ __forceinline__ void operator()() const {}
};

template <int F, int T>
__global__ void __launch_bounds__(PassShape<F, T>::NT, 3) fft_pass_rdb_kernel(const PassDesc d, int64_t tiles) {
    extern __shared__ double2 sm[];
    double2 *tw = reinterpret_cast<double2 *>(reinterpret_cast<char *>(sm) + PassShape<F, T>::XCH);
    const TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    int64_t tile = blockIdx.x;
    if (tile >= tiles) return;
    double2 nx[PassShape<F, T>::R];
    rdb_load_tile<F, T>(nx, d, io, tile);
    for (; tile < tiles; tile += gridDim.x) {
        const RdbHook<F, T> hk{nx, &d, &io, tile + (int64_t)gridDim.x, tiles};
        tile_fft<F, T, 6, RdbHook<F, T>>(sm, tw, d, io, tile, nullptr, hk);
        __syncthreads();   // every lane is done with the exchange buffer and the tables
    }
}

template <int F, int T>
cudaError_t launch_one_rdb(const PassDesc &d, int64_t tiles, int grid, cudaStream_t s) {
    using SH = PassShape<F, T>;
    fft_pass_rdb_kernel<F, T><<<grid, SH::NT, SH::SMEM, s>>>(d, tiles);
    return cudaGetLastError();
}

template <int F, int T>
int grid_one_rdb() {
    using SH = PassShape<F, T>;
    if (SH::SMEM > 48 * 1024 &&
        cudaFuncSetAttribute(fft_pass_rdb_kernel<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::SMEM) !=
            cudaSuccess)
        return 0;
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft_pass_rdb_kernel<F, T>, SH::NT, SH::SMEM) !=
        cudaSuccess)
        return 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}

// persistent plain pass: the tile loop of fft_pass_kernel without CTA turnover
template <int F, int T>
__global__ void __launch_bounds__(PassShape<F, T>::NT, PassShape<F, T>::MINB)
    fft_pass_persist_kernel(const PassDesc d, int64_t tiles) {
    extern __shared__ double2 sm[];
    double2 *tw = reinterpret_cast<double2 *>(reinterpret_cast<char *>(sm) + PassShape<F, T>::XCH);
    const TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        __syncthreads();   // the previous tile is done with the exchange buffer and the tables
        tile_fft<F, T>(sm, tw, d, io, tile);
    }
}

template <int F, int T>
cudaError_t launch_one_pf(const PassDesc &d, int64_t tiles, int grid, cudaStream_t s) {
    using SH = PassShape<F, T>;
    static const int pf_kind = [] {
        const char *e = getenv("MOA_FFT_PF");
        return e ? atoi(e) : 0;
    }();
    if (pf_kind == 3) return launch_one_rdb<F, T>(d, tiles, grid, s);
    if (pf_kind == 2) {
        if (SH::SMEM > 48 * 1024)
            cudaFuncSetAttribute(fft_pass_persist_kernel<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SH::SMEM);
        fft_pass_persist_kernel<F, T><<<grid, SH::NT, SH::SMEM, s>>>(d, tiles);
    } else {
        fft_pass_pf_kernel<F, T><<<grid, SH::NT, SH::SMEM, s>>>(d, tiles);
    }
    return cudaGetLastError();
}

template <int F, int T>
int grid_one_pf() {
    using SH = PassShape<F, T>;
    const char *e = getenv("MOA_FFT_PF");
    if (e && atoi(e) == 3) return grid_one_rdb<F, T>();
    if (SH::SMEM > 48 * 1024 &&
        cudaFuncSetAttribute(fft_pass_pf_kernel<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::SMEM) !=
            cudaSuccess)
        return 0;
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft_pass_pf_kernel<F, T>, SH::NT, SH::SMEM) !=
        cudaSuccess)
        return 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}

#endif  // MOA_VARIANTS

template <int F, int T>
cudaError_t launch_one(const PassDesc &d, int64_t tiles, cudaStream_t s) {
    using SH = PassShape<F, T>;
    auto kernel = d.twiddle ? fft_pass_kernel<F, T, 1> : fft_pass_kernel<F, T, 0>;
    if (d.pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)tiles);
        cfg.blockDim = dim3(SH::NT);
        cfg.dynamicSmemBytes = SH::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kernel, d);
    }
    kernel<<<(unsigned)tiles, SH::NT, SH::SMEM, s>>>(d);
    return cudaGetLastError();
}

template <int F, int T>
cudaError_t prepare_one() {
    using SH = PassShape<F, T>;
    if (SH::SMEM > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fft_pass_kernel<F, T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)SH::SMEM);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fft_pass_kernel<F, T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::SMEM);
        if (e != cudaSuccess) return e;
        if constexpr (F >= 256 && T <= 16) {   // the bulk-tensor-store row pass (launch_tmast)
            e = cudaFuncSetAttribute(fft_pass_tmast_kernel<F, T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)SH::SMEM);
            if (e != cudaSuccess) return e;
            return cudaFuncSetAttribute(fft_pass_tmast_kernel<F, T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)SH::SMEM);
        }
    }
    return cudaSuccess;
}

}  // namespace moa

#ifdef MOA_VARIANTS
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
    // one buffer = the TMA staging tile, reused in place as the exchange buffer
    static constexpr size_t BUF = ((IN_BYTES > PassShape<F, T>::XCH ? IN_BYTES : PassShape<F, T>::XCH) + 127) / 128 * 128;
    static constexpr size_t TW = PassShape<F, T>::TWA + PassShape<F, T>::TWB;
    static constexpr size_t SMEM = 128 + 2 * BUF + TW + 32;
};

template <int F, int T, int SRC>
__device__ __forceinline__ void tma_issue_tile(const CUtensorMap *map, uint64_t *bar, double2 *inbuf,
                                               const PassDesc &d, int64_t tile) {
    using TS = TmaShape<F, T, SRC>;
    const int u = (int)(tile & (d.U - 1));
    const int v = (int)((tile >> d.lU) & (d.V - 1));
    const int w = (int)(tile >> (d.lU + d.lV));
    mbar_expect_tx(bar, TS::BOX_BYTES * TS::NBOX);
#pragma unroll
    for (int k = 0; k < TS::NBOX; ++k) {
        if constexpr (SRC == 1)   // column tile: dims {2B doubles, F, A}
            tma_load_3d(inbuf + k * TS::FB * T, map, bar, 2 * T * u, k * TS::FB, v);
        else                      // row tile: dims {2F doubles, rows, V, W}
            tma_load_4d(inbuf + k * TS::FB * T, map, bar, 2 * TS::FB * k, T * u, v, w);
    }
}

struct SyncHook {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

#ifndef MOA_TMA_MINB
#define MOA_TMA_MINB 3
#endif
// Persistent TMA pass, double buffered: while tile i is transformed in buffer
// i&1 (staged input, then reused in place for the exchanges), the copy of tile
// i+1 streams into the other buffer.
template <int F, int T, int SRC>
__global__ void __launch_bounds__(PassShape<F, T>::NT, (T * F <= 2048) ? MOA_TMA_MINB : 1)
    fft_pass_tma_kernel(const PassDesc d, const __grid_constant__ CUtensorMap tmap, int64_t tiles) {
    using TS = TmaShape<F, T, SRC>;
    extern __shared__ unsigned char smraw[];
    // align by pointer arithmetic (an integer round trip would lose the shared
    // address space and turn every exchange access into a generic LD/ST)
    unsigned char *base = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
    auto buf = [&](int i) { return reinterpret_cast<double2 *>(base + i * TS::BUF); };
    double2 *tw = reinterpret_cast<double2 *>(base + 2 * TS::BUF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(base + 2 * TS::BUF + TS::TW);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    int64_t tile = blockIdx.x;
    if (tid == 0 && tile < tiles) tma_issue_tile<F, T, SRC>(&tmap, &bar[0], buf(0), d, tile);
    const TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    for (int it = 0; tile < tiles; tile += gridDim.x, ++it) {
        const int b = it & 1;
        __syncthreads();   // the previous tile is done with buf(b^1) and the twiddle tables
        const int64_t next = tile + gridDim.x;
        if (tid == 0 && next < tiles) {
            fence_proxy_async();
            tma_issue_tile<F, T, SRC>(&tmap, &bar[b ^ 1], buf(b ^ 1), d, next);
        }
        mbar_wait(&bar[b], (it >> 1) & 1);
        tile_fft<F, T, SRC, SyncHook>(buf(b), tw, d, io, tile, buf(b), SyncHook());
    }
}

// ---------------------------------------------------------------------------
// Persistent TMA pass with ONE staging buffer per CTA (SRC 4 = column tile, 5 = row
// tile): the tile arrives by cp.async.bulk.tensor into the buffer that later holds the
// shared-memory exchange; as soon as the last butterfly stage has read the exchange,
// one elected thread starts the bulk copy of the CTA's next tile into the same buffer,
// so that copy overlaps the last butterflies, the twiddles and the stores.  Same
// shared memory as fft_pass_kernel (4 CTAs/SM at F*T = 2048); no per-thread copy
// instructions (the cp.async variant flooded the MIO queue).
template <int F, int T, int SRC>
struct TpfShape {
    static constexpr int SLAY = SRC == 4 ? 1 : 2;
    using TS = TmaShape<F, T, SLAY>;
    static constexpr size_t BUF = ((TS::IN_BYTES > PassShape<F, T>::XCH ? TS::IN_BYTES : PassShape<F, T>::XCH) + 127) / 128 * 128;
    static constexpr size_t TW = PassShape<F, T>::TWA + PassShape<F, T>::TWB;
    static constexpr size_t SMEM = 128 + BUF + TW + 16;
};

template <int F, int T, int SRC>
struct TpfHook {
    const CUtensorMap *map;
    uint64_t *bar;
    double2 *buf;
    const PassDesc *d;
    int64_t next, tiles;
    __device__ __forceinline__ void operator()() const {
        __syncthreads();   // every lane has read the exchange buffer
        if (threadIdx.x == 0 && next < tiles) {
            fence_proxy_async();   // the generic-proxy reads are ordered before the async writes
            tma_issue_tile<F, T, TpfShape<F, T, SRC>::SLAY>(map, bar, buf, *d, next);
        }
    }
};

template <int F, int T, int SRC>
__global__ void __launch_bounds__(PassShape<F, T>::NT, PassShape<F, T>::MINB)
    fft_pass_tpf_kernel(const PassDesc d, const __grid_constant__ CUtensorMap tmap, int64_t tiles) {
    using SH = TpfShape<F, T, SRC>;
    extern __shared__ unsigned char smraw[];
    unsigned char *base = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
    double2 *buf = reinterpret_cast<double2 *>(base);
    double2 *tw = reinterpret_cast<double2 *>(base + SH::BUF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(base + SH::BUF + SH::TW);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    int64_t tile = blockIdx.x;
    if (tile >= tiles) return;
    if (threadIdx.x == 0) tma_issue_tile<F, T, SH::SLAY>(&tmap, bar, buf, d, tile);
    const TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    for (int it = 0; tile < tiles; tile += gridDim.x, ++it) {
        mbar_wait(bar, it & 1);
        const TpfHook<F, T, SRC> hk{&tmap, bar, buf, &d, tile + (int64_t)gridDim.x, tiles};
        tile_fft<F, T, SRC, TpfHook<F, T, SRC>>(buf, tw, d, io, tile, buf, hk);
        __syncthreads();   // the epilogue is done with the twiddle tables
    }
}

// ---------------------------------------------------------------------------
// Non-persistent TMA-loaded pass (SRC 6 = column tile, 7 = row tile): the plain pass's
// one tile per CTA, but the tile arrives as ONE bulk-tensor copy issued by one thread
// (box {2T doubles, 256 points} or row boxes) into the exchange buffer under an
// mbarrier instead of 16 LDG.128 per thread; the first stage reads it from shared memory
// and the buffer becomes the exchange buffer.  Same shared memory and occupancy as
// fft_pass_kernel.
template <int F, int T, int SRC>
__global__ void __launch_bounds__(PassShape<F, T>::NT, PassShape<F, T>::MINB)
    fft_pass_tma1_kernel(const PassDesc d, const __grid_constant__ CUtensorMap tmap) {
    constexpr int SL = SRC == 6 ? 1 : 2;
    using SH = TpfShape<F, T, SL + 3>;
    extern __shared__ unsigned char smraw[];
    unsigned char *base = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
    double2 *buf = reinterpret_cast<double2 *>(base);
    double2 *tw = reinterpret_cast<double2 *>(base + SH::BUF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(base + SH::BUF + SH::TW);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (d.pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) tma_issue_tile<F, T, SL>(&tmap, bar, buf, d, blockIdx.x);
    const TileIO io{d.src, d.dst, d.in_shift, d.out_shift};
    mbar_wait(bar, 0);
    tile_fft<F, T, SL, SyncHook>(buf, tw, d, io, blockIdx.x, buf, SyncHook());
}

template <int F, int T, int SRC>
cudaError_t launch_one_tma1(const PassDesc &d, const CUtensorMap &map, int64_t tiles, cudaStream_t s) {
    using SH = TpfShape<F, T, (SRC == 6 ? 1 : 2) + 3>;
    static_assert(SH::SMEM <= 227 * 1024, "smem");
    if (SH::SMEM > 48 * 1024)
        cudaFuncSetAttribute(fft_pass_tma1_kernel<F, T, SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SH::SMEM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tiles);
    cfg.blockDim = dim3(PassShape<F, T>::NT);
    cfg.dynamicSmemBytes = SH::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = d.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fft_pass_tma1_kernel<F, T, SRC>, d, map);
}

template <int F, int T, int SRC>
cudaError_t launch_one_tpf(const PassDesc &d, const CUtensorMap &map, int64_t tiles, int grid, cudaStream_t s) {
    fft_pass_tpf_kernel<F, T, SRC><<<grid, PassShape<F, T>::NT, TpfShape<F, T, SRC>::SMEM, s>>>(d, map, tiles);
    return cudaGetLastError();
}

template <int F, int T, int SRC>
int grid_one_tpf() {
    using SH = TpfShape<F, T, SRC>;
    if (SH::SMEM > 48 * 1024 &&
        cudaFuncSetAttribute(fft_pass_tpf_kernel<F, T, SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SH::SMEM) != cudaSuccess)
        return 0;
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft_pass_tpf_kernel<F, T, SRC>, PassShape<F, T>::NT,
                                                      SH::SMEM) != cudaSuccess)
        return 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
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
#endif  // MOA_VARIANTS
