// bigpass.cu -- the 4096-point lifted pass as a persistent, TMA-fed kernel (SURVEY §8(a)
// S3/S4 for liftings <4096, 4096> and friends: two HBM passes at n = 2^24 instead of three).
//
// The paper's lifting lets each level be any size the memory hierarchy holds ("any
// partition size", "not necessarily blocked in squares") and hides the cost of the
// periodic rearrangement by prefetching.  On B200 a 4096-point level of T = 2
// columns is a 128 KiB tile: the whole register file of one SM (512 threads x 16 points).
// One CTA per SM therefore cannot overlap its own load, butterflies and store the way
// four small CTAs do -- unless the load of tile i+1 is issued to the TMA engine before
// tile i's butterflies start:
//
//   shared memory: S = staging for the NEXT tile (128 KiB, written by cp.async.bulk[.tensor]
//                  under an mbarrier), X = exchange buffer (64 KiB: half of the positions
//                  of both transforms at a time), B = per-tile output-twiddle table
//   per tile:      wait(mbarrier) -> 16 points per thread from S -> barrier -> one thread
//                  issues the TMA copy of the CTA's next tile into S -> three radix-16
//                  Stockham stages (Fig 3.7 butterflies grouped by 16; DFT_16 in registers)
//                  with two exchanges through X -> twiddle -> 16 stores per thread
//
// Column tiles (middle pass, view [A][4096][B]) arrive by a 3-D bulk-tensor copy of
// 16 boxes {2 columns, 256 points}; row tiles (last pass) by two 64 KiB bulk copies.
// Each exchange runs in two rounds of 2048 positions per transform (X is half a tile):
// exchange 1 splits positions by bit 3 ^ bit 11 (slot = p without bit 11), exchange 2 by
// bit 4 ^ bit 8 (slot = p without bit 8), so every thread writes 8 and reads 8 values per
// round -- the same 8 registers on both sides, with a warp-uniform round choice -- and
// the addresses t*2048 + (q ^ swz(q) ^ 5t) are conflict-free for all four exchange
// accesses (tools/bank_sim_big.py).
//
// Measured slower than three 256-point passes (2^24: 346 vs 260 µs; DESIGN.md §11,
// profiles/r02_two_pass_2e24.md): compiled only into libmoa_fft_variants.so.
#include "fft_pass.cuh"

namespace moa {

namespace big {

constexpr int F = 4096;       // points per transform
constexpr int T = 2;          // transforms per tile
constexpr int NT = 512;       // threads: 16 points each
constexpr int NB = F / 16;    // butterflies per transform and stage
constexpr int S_ROW = F + 4;  // row tiles: transform t staged at S + t*S_ROW (bank offset 4)
constexpr size_t S_BYTES = (size_t)(S_ROW + F) * 16;  // 128 KiB (+64 B) staging
constexpr size_t X_BYTES = (size_t)T * (F / 2) * 16;  // 64 KiB exchange
constexpr size_t B_BYTES = (size_t)T * 16 * 16;       // output twiddles omega^(beta_t*256*r)
constexpr size_t W_BYTES = (size_t)(256 + NT) * 16;     // omega_256^m (stage 2), omega_4096^j per thread (stage 3)
constexpr size_t SMEM = 128 + S_BYTES + X_BYTES + B_BYTES + W_BYTES + 16;

__host__ __device__ constexpr int swz3(int q) { return ((q >> 3) ^ (q >> 6) ^ (q >> 9)) & 7; }

// exchange slot of position p (0..4095) of transform t within its round: p with bit
// DROP removed, bank-group swizzled (tools/bank_sim_big.py)
template <int DROP>
__device__ __forceinline__ int xaddr(int t, int p) {
    const int q = (p & ((1 << DROP) - 1)) | ((p >> (DROP + 1)) << DROP);
    return t * (F / 2) + (q ^ swz3(q) ^ (5 * t));
}

// write / read the values r whose bit RB equals B, at positions pbase + STRIDE*r
template <int B, int RB, int STRIDE, int DROP>
__device__ __forceinline__ void xw8(double2 *X, const double2 *x, int t, int pbase) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if (((r >> RB) & 1) == B) X[xaddr<DROP>(t, pbase + STRIDE * r)] = x[r];
}
template <int B, int RB, int STRIDE, int DROP>
__device__ __forceinline__ void xr8(const double2 *X, double2 *x, int t, int pbase) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if (((r >> RB) & 1) == B) x[r] = X[xaddr<DROP>(t, pbase + STRIDE * r)];
}

// One Stockham exchange in two rounds through the half-tile buffer X.  The writer's 16
// values go to positions pw + WS*r, the reader's come from pr + RS*r (same transform t).
// Round R moves the values r with bit RB of r equal to s ^ R on BOTH sides (the lane
// maps make the write and read register sets of a round identical, and s warp-uniform):
// each round writes 8 registers, then refills the same 8, so 16 values stay live.
template <int WS, int RS, int RB, int DROP>
__device__ __forceinline__ void exchange(double2 *X, double2 *x, int t, int pw, int pr, int s) {
    __syncthreads();   // the previous readers of X are done
    if (s) xw8<1, RB, WS, DROP>(X, x, t, pw); else xw8<0, RB, WS, DROP>(X, x, t, pw);
    __syncthreads();
    if (s) xr8<1, RB, RS, DROP>(X, x, t, pr); else xr8<0, RB, RS, DROP>(X, x, t, pr);
    __syncthreads();
    if (s) xw8<0, RB, WS, DROP>(X, x, t, pw); else xw8<1, RB, WS, DROP>(X, x, t, pw);
    __syncthreads();
    if (s) xr8<0, RB, RS, DROP>(X, x, t, pr); else xr8<1, RB, RS, DROP>(X, x, t, pr);
}

// stage twiddles x[s] *= w^s (s = 0..15) from w, w^2, w^4, w^8, optionally with the pass
// twiddle's common factor a folded in (x[s] *= a * w^s): the power chain of
// stage_twiddle / stage_twiddle_scaled (fft_pass.cuh) with the four bases as values
template <bool SCALED>
__device__ __forceinline__ void stw16(double2 *x, double2 w1, double2 w2, double2 w4, double2 w8, double2 a) {
    double2 c1 = w1, c2 = w2, c4 = w4, c8 = w8;
    if constexpr (SCALED) {
        x[0] = cmul(x[0], a);
        c1 = cmul(a, w1);
        c2 = cmul(a, w2);
        c4 = cmul(a, w4);
        c8 = cmul(a, w8);
    }
    const double2 c3 = cmul(c1, w2);
    x[1] = cmul(x[1], c1);
    x[2] = cmul(x[2], c2);
    x[3] = cmul(x[3], c3);
    const double2 c5 = cmul(c1, w4), c6 = cmul(c2, w4), c7 = cmul(c3, w4);
    x[4] = cmul(x[4], c4);
    x[5] = cmul(x[5], c5);
    x[6] = cmul(x[6], c6);
    x[7] = cmul(x[7], c7);
    x[8] = cmul(x[8], c8);
    x[9] = cmul(x[9], cmul(c1, w8));
    x[10] = cmul(x[10], cmul(c2, w8));
    x[11] = cmul(x[11], cmul(c3, w8));
    x[12] = cmul(x[12], cmul(c4, w8));
    x[13] = cmul(x[13], cmul(c5, w8));
    x[14] = cmul(x[14], cmul(c6, w8));
    x[15] = cmul(x[15], cmul(c7, w8));
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// tile id -> (u, v, w) (PassDesc convention)
struct TileIdx {
    int64_t u, v, w;
    __device__ __forceinline__ TileIdx(const PassDesc &d, int64_t b) {
        u = b & (d.U - 1);
        v = (b >> d.lU) & (d.V - 1);
        w = b >> (d.lU + d.lV);
    }
};

// issue the copy of `tile` into S (one thread)
template <int ROW>
__device__ __forceinline__ void issue_tile(const PassDesc &d, const CUtensorMap *map, uint64_t *bar, double2 *S,
                                           int64_t tile) {
    const TileIdx ti(d, tile);
    mbar_expect_tx(bar, (unsigned)(F * T * 16));
    if constexpr (ROW) {   // two contiguous rows of F points
        const double2 *src = d.src + (ti.u * d.in_u + ti.v * d.in_v + ti.w * d.in_w);
#pragma unroll
        for (int t = 0; t < T; ++t) bulk_load(S + t * S_ROW, src + t * d.in_t, (uint32_t)(F * 16), bar);
    } else {               // 16 boxes {2 columns, 256 points}: S[f][t]
#pragma unroll
        for (int k = 0; k < F / 256; ++k) tma_load_3d(S + k * 256 * T, map, bar, (int)(2 * T * ti.u), k * 256, (int)ti.v);
    }
}

// ROW = 1: last pass (rows of F contiguous points, output through the out_* map);
// ROW = 0: middle pass (column tile of the view [A][F][B], stored in place).
// TW: the pass multiplies output k of transform t by omega_n^(alpha_t + beta_t*k).
template <int ROW, int TW>
__global__ void __launch_bounds__(NT, 1) fft4096_kernel(const PassDesc d, const __grid_constant__ CUtensorMap map,
                                                        int64_t tiles) {
    extern __shared__ unsigned char smraw[];
    unsigned char *base = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
    double2 *S = reinterpret_cast<double2 *>(base);
    double2 *X = reinterpret_cast<double2 *>(base + S_BYTES);
    double2 *TB = reinterpret_cast<double2 *>(base + S_BYTES + X_BYTES);
    double2 *W2 = reinterpret_cast<double2 *>(base + S_BYTES + X_BYTES + B_BYTES);   // [256]
    double2 *W3 = W2 + 256;                                                             // [NT]
    uint64_t *bar = reinterpret_cast<uint64_t *>(base + S_BYTES + X_BYTES + B_BYTES + W_BYTES);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (d.pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    __syncthreads();
    int64_t tile = blockIdx.x;
    if (tid == 0 && tile < tiles) issue_tile<ROW>(d, &map, bar, S, tile);

    // lane maps (tools/bank_sim_big.py): transform t = tid & 1 in every stage; stages 1
    // and 3 take butterfly j = tid >> 1 (stage 3 then stores 32-byte runs: lanes t = 0, 1
    // write adjacent columns), stage 2 a permutation of it that makes both exchanges'
    // round choices (s1 = tid bit 8, s2 = tid bit 5) agree on the writer and reader side
    const int t0 = tid & 1, j130 = tid >> 1;
    const int j20 = ((tid >> 1) & 7) | (((tid >> 8) & 1) << 3) | (((tid >> 5) & 1) << 4) | (((tid >> 4) & 1) << 5) |
                    (((tid >> 6) & 1) << 6) | (((tid >> 7) & 1) << 7);
    const uint32_t nm = (uint32_t)d.nmask;
    // the stage twiddles are the same for every tile: stage 2 reads omega_256^m from a
    // shared table, stage 3 this thread's omega_4096^j (then squares it): no global loads
    // on the per-tile critical path
    if (tid < 256) W2[tid] = d.tw_f[tid * (FMAX / 256)];
    W3[tid] = d.tw_f[j130 * (FMAX / F)];

    for (int it = 0; tile < tiles; tile += gridDim.x, ++it) {
        // re-derive the lane indices every tile (opaque to the compiler): otherwise it
        // hoists the 64 loop-invariant exchange addresses out of the tile loop and spills
        int t = t0, j13 = j130, j2 = j20;
        asm volatile("" : "+r"(t), "+r"(j13), "+r"(j2));
        const int s1 = (j13 >> 7) & 1, s2 = (j13 >> 4) & 1;
        const TileIdx ti(d, tile);
        double2 x[16];
        mbar_wait(bar, (unsigned)(it & 1));
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = ROW ? S[t * S_ROW + j13 + NB * r] : S[(j13 + NB * r) * T + t];
        if (d.conj_in) {
#pragma unroll
            for (int r = 0; r < 16; ++r) x[r].y = -x[r].y;
        }
        // output address of point k = j + 256 r of transform t: po + r * so
        double2 *const po = d.dst + (ti.u * d.out_u + ti.v * d.out_v + ti.w * d.out_w - d.out_shift) +
                            t * d.out_t + (int64_t)j13 * d.out_k;
        __syncthreads();   // every lane has read S (and the previous tile's B table)
        if (tid == 0 && tile + gridDim.x < tiles) {
            fence_proxy_async();   // generic-proxy reads of S before the async-proxy writes
            issue_tile<ROW>(d, &map, bar, S, tile + gridDim.x);
        }
        uint32_t al = 0, be = 0;
        if constexpr (TW) {
            al = (uint32_t)d.a_c + (uint32_t)ti.u * (uint32_t)d.a_u + (uint32_t)ti.v * (uint32_t)d.a_v +
                 (uint32_t)ti.w * (uint32_t)d.a_w;
            be = (uint32_t)d.b_c + (uint32_t)ti.u * (uint32_t)d.b_u + (uint32_t)ti.v * (uint32_t)d.b_v +
                 (uint32_t)ti.w * (uint32_t)d.b_w;
            if (tid < T * 16) {   // B[t][r] = omega_n^(beta_t * 256 * r)
                const int t = tid >> 4, r = tid & 15;
                const uint32_t bt = be + (uint32_t)t * (uint32_t)d.b_t;
                TB[tid] = root_pi((bt * (uint32_t)(NB * r)) & nm, d.tbits);
            }
        }
        // stage 1 (NS = 1): DFT_16 of points j + 256 r -> positions 16 j + r
        dft_reg<16>(x);
        exchange<1, NB, 3, 11>(X, x, t, 16 * j13, j2, s1);
        // stage 2 (NS = 16): twiddle omega_256^((j2 % 16) r), DFT_16 -> (j2/16)*256 + j2%16 + 16 r
        {
            const int e = j2 & 15;
            stw16<false>(x, W2[e], W2[2 * e], W2[4 * e], W2[8 * e], make_double2(1.0, 0.0));
        }
        dft_reg<16>(x);
        exchange<16, NB, 0, 8>(X, x, t, (j2 >> 4) * 256 + (j2 & 15), j13, s2);
        // stage 3 (NS = 256): twiddle omega_4096^(j3 r) (with the pass twiddle's factor
        // omega_n^(alpha_t + beta_t j3) folded in), DFT_16 -> output k = j3 + 256 r
        if constexpr (TW) {
            const uint32_t at = al + (uint32_t)t * (uint32_t)d.a_t, bt = be + (uint32_t)t * (uint32_t)d.b_t;
            const double2 a = root_pi((at + bt * (uint32_t)j13) & nm, d.tbits);
            const double2 w1 = W3[tid], w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
            stw16<true>(x, w1, w2, w4, w8, a);
            dft_reg<16>(x);
#pragma unroll
            for (int r = 1; r < 16; ++r) x[r] = cmul(x[r], TB[t * 16 + r]);
        } else {
            const double2 w1 = W3[tid], w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
            stw16<false>(x, w1, w2, w4, w8, make_double2(1.0, 0.0));
            dft_reg<16>(x);
        }
        if (d.conj_out) {
#pragma unroll
            for (int r = 0; r < 16; ++r) x[r].y = -x[r].y;
        }
        const int64_t so = (int64_t)NB * d.out_k;
#pragma unroll
        for (int r = 0; r < 16; ++r)
            asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(po + r * so), "d"(x[r].x), "d"(x[r].y) : "memory");
    }
}

}  // namespace big

// ------------------------------------------------------------------ host side
int big_supported(int logF, int T) { return logF == 12 && T == big::T; }

size_t big_smem_bytes() { return big::SMEM; }

cudaError_t prepare_big_kernels() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(big::fft4096_kernel<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)big::SMEM)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(big::fft4096_kernel<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)big::SMEM)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(big::fft4096_kernel<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)big::SMEM)) != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(big::fft4096_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)big::SMEM);
}

cudaError_t launch_big(const PassDesc &d, const CUtensorMap &map, int64_t tiles, cudaStream_t s) {
    const int row = d.in_f == 1;
    auto kernel = row ? (d.twiddle ? big::fft4096_kernel<1, 1> : big::fft4096_kernel<1, 0>)
                      : (d.twiddle ? big::fft4096_kernel<0, 1> : big::fft4096_kernel<0, 0>);
    const int64_t sms = sm_count();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(tiles < sms ? tiles : sms));
    cfg.blockDim = dim3(big::NT);
    cfg.dynamicSmemBytes = big::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = d.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, d, map, tiles);
}

}  // namespace moa
