// kernels.cu -- the non-lifted kernels and the pass dispatcher.
//   K1 bitrev          P_n of Fig 2.1 line 1          [literal mode]
//   K2 radix2_stage    one q-stage of Fig 3.9              [literal mode]
//   K6 pcombine<P>     the cyclic phase q = breakpoint..t of Fig 5.7 in
//                      its lifted form: a P-point DFT across the received chunks
//   gen_uniform        the SplitMix64 input recipe (test/bench helper, no FFT arithmetic)
#include "fft_pass.cuh"

#include <atomic>

namespace moa {

// SM count of the current device (queried once per device, then cached)
int sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev].load() <= 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 1;
        }
        cache[dev].store(v);
    }
    return cache[dev].load();
}

// ------------------------------------------------------------------ dispatcher
int pass_supported(int logF, int T) {
    if (logF < 1 || logF > FMAX_LOG) return 0;
    if (T < 1 || T > 64 || (T & (T - 1))) return 0;
    return ((int64_t)T << logF) <= TF_MAX;
}

int pass_threads(int logF, int T) {
    int F = 1 << logF;
    int R = F >= MOA_RMAX ? MOA_RMAX : F;
    return T * F / R;
}

size_t pass_smem_bytes(int logF, int T) {
    int F = 1 << logF;
    if (F <= 16) return 0;
    int pad = T == 1 ? 0 : (T == 2 ? 4 : (T == 4 ? 2 : 1));
    return (size_t)T * (F + pad) * sizeof(double2);
}

cudaError_t launch_pass(int logF, int T, const PassDesc &d, int64_t tiles, cudaStream_t s) {
    if (!pass_supported(logF, T) || tiles <= 0 || tiles > 0x7fffffffll) return cudaErrorInvalidValue;
    switch (logF) {
    case 1: return launch_pass_f1(T, d, tiles, s);
    case 2: return launch_pass_f2(T, d, tiles, s);
    case 3: return launch_pass_f3(T, d, tiles, s);
    case 4: return launch_pass_f4(T, d, tiles, s);
    case 5: return launch_pass_f5(T, d, tiles, s);
    case 6: return launch_pass_f6(T, d, tiles, s);
    case 7: return launch_pass_f7(T, d, tiles, s);
    case 8: return launch_pass_f8(T, d, tiles, s);
    case 9: return launch_pass_f9(T, d, tiles, s);
    case 10: return launch_pass_f10(T, d, tiles, s);
    case 11: return launch_pass_f11(T, d, tiles, s);
    case 12: return launch_pass_f12(T, d, tiles, s);
    case 13: return launch_pass_f13(T, d, tiles, s);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_pass_tmast(int logF, int T, const PassDesc &d, const CUtensorMap &omap, int64_t tiles,
                              cudaStream_t s) {
    if (tiles <= 0 || tiles > 0x7fffffffll) return cudaErrorInvalidValue;
    switch (logF) {
    case 8: return launch_pass_tmast_f8(T, d, omap, tiles, s);
    case 9: return launch_pass_tmast_f9(T, d, omap, tiles, s);
    case 10: return launch_pass_tmast_f10(T, d, omap, tiles, s);
    case 11: return launch_pass_tmast_f11(T, d, omap, tiles, s);
    case 12: return launch_pass_tmast_f12(T, d, omap, tiles, s);
    case 13: return launch_pass_tmast_f13(T, d, omap, tiles, s);
    default: return cudaErrorInvalidValue;
    }
}

#ifdef MOA_VARIANTS
int pass_tma_grid(int logF, int T, int src) {
    switch (logF) {
    case 5: return grid_pass_tma_f5(T, src);
    case 6: return grid_pass_tma_f6(T, src);
    case 7: return grid_pass_tma_f7(T, src);
    case 8: return grid_pass_tma_f8(T, src);
    case 9: return grid_pass_tma_f9(T, src);
    case 10: return grid_pass_tma_f10(T, src);
    case 11: return grid_pass_tma_f11(T, src);
    case 12: return grid_pass_tma_f12(T, src);
    default: return 0;
    }
}

cudaError_t launch_pass_tma(int logF, int T, int src, const PassDesc &d, const CUtensorMap &map, int64_t tiles,
                            int grid, cudaStream_t s) {
    switch (logF) {
    case 5: return launch_pass_tma_f5(T, src, d, map, tiles, grid, s);
    case 6: return launch_pass_tma_f6(T, src, d, map, tiles, grid, s);
    case 7: return launch_pass_tma_f7(T, src, d, map, tiles, grid, s);
    case 8: return launch_pass_tma_f8(T, src, d, map, tiles, grid, s);
    case 9: return launch_pass_tma_f9(T, src, d, map, tiles, grid, s);
    case 10: return launch_pass_tma_f10(T, src, d, map, tiles, grid, s);
    case 11: return launch_pass_tma_f11(T, src, d, map, tiles, grid, s);
    case 12: return launch_pass_tma_f12(T, src, d, map, tiles, grid, s);
    default: return cudaErrorInvalidValue;
    }
}

int pass_pf_grid(int logF, int T) {
    switch (logF) {
    case 5: return grid_pass_pf_f5(T);
    case 6: return grid_pass_pf_f6(T);
    case 7: return grid_pass_pf_f7(T);
    case 8: return grid_pass_pf_f8(T);
    case 9: return grid_pass_pf_f9(T);
    case 10: return grid_pass_pf_f10(T);
    case 11: return grid_pass_pf_f11(T);
    case 12: return grid_pass_pf_f12(T);
    case 13: return grid_pass_pf_f13(T);
    default: return 0;
    }
}

cudaError_t launch_pass_pf(int logF, int T, const PassDesc &d, int64_t tiles, int grid, cudaStream_t s) {
    switch (logF) {
    case 5: return launch_pass_pf_f5(T, d, tiles, grid, s);
    case 6: return launch_pass_pf_f6(T, d, tiles, grid, s);
    case 7: return launch_pass_pf_f7(T, d, tiles, grid, s);
    case 8: return launch_pass_pf_f8(T, d, tiles, grid, s);
    case 9: return launch_pass_pf_f9(T, d, tiles, grid, s);
    case 10: return launch_pass_pf_f10(T, d, tiles, grid, s);
    case 11: return launch_pass_pf_f11(T, d, tiles, grid, s);
    case 12: return launch_pass_pf_f12(T, d, tiles, grid, s);
    case 13: return launch_pass_pf_f13(T, d, tiles, grid, s);
    default: return cudaErrorInvalidValue;
    }
}

#else
// product build: the persistent / TMA-staged / prefetching pass variants and the
// L2-fused pass pair were measured slower and are compiled only into
// libmoa_fft_variants.so (MOA_BUILD_VARIANTS=1); the plan never selects them here
int pass_tma_grid(int, int, int) { return 0; }
cudaError_t launch_pass_tma(int, int, int, const PassDesc &, const CUtensorMap &, int64_t, int, cudaStream_t) {
    return cudaErrorInvalidValue;
}
int pass_pf_grid(int, int) { return 0; }
cudaError_t launch_pass_pf(int, int, const PassDesc &, int64_t, int, cudaStream_t) { return cudaErrorInvalidValue; }
int fused_supported(int, int, int, int) { return 0; }
cudaError_t launch_fused(int, int, int, int, const FusedDesc &, const CUtensorMap &, const CUtensorMap &, int,
                         cudaStream_t) {
    return cudaErrorInvalidValue;
}
int fused_grid(int, int, int, int) { return 0; }
int big_supported(int, int) { return 0; }
cudaError_t prepare_big_kernels() { return cudaSuccess; }
cudaError_t launch_big(const PassDesc &, const CUtensorMap &, int64_t, cudaStream_t) { return cudaErrorInvalidValue; }
#endif

cudaError_t prepare_pass_kernels() {
    cudaError_t (*fns[])() = {prepare_pass_f1, prepare_pass_f2, prepare_pass_f3, prepare_pass_f4,
                              prepare_pass_f5, prepare_pass_f6, prepare_pass_f7, prepare_pass_f8,
                              prepare_pass_f9, prepare_pass_f10, prepare_pass_f11, prepare_pass_f12,
                              prepare_pass_f13};
    for (auto f : fns) {
        cudaError_t e = f();
        if (e != cudaSuccess) return e;
    }
    return prepare_big_kernels();
}

// ------------------------------------------------------------------ K1: bit reversal
__device__ __forceinline__ uint64_t rev_bits(uint64_t j, int t) { return __brevll(j) >> (64 - t); }

// y[j] = x[rev_t(j)], small t: one thread per output (reads are a permutation).
__global__ void bitrev_direct(const double2 *__restrict__ x, double2 *__restrict__ y, int t, int conj_in) {
    uint64_t n = 1ull << t;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
         j += (uint64_t)gridDim.x * blockDim.x) {
        double2 v = x[rev_bits(j, t)];
        if (conj_in) v.y = -v.y;
        y[j] = v;
    }
}

// t >= 10: j = (a | m | b) with 5-bit a, b: rev(j) = (rev5 b | rev m | rev5 a).
// A 32x32 tile per middle value m, so both the reads and the writes are
// 512-byte contiguous runs.
__global__ void __launch_bounds__(256) bitrev_tiled(const double2 *__restrict__ x, double2 *__restrict__ y,
                                                     int t, int conj_in) {
    __shared__ double2 tile[32][33];
    const int mb = t - 10;
    const uint64_t m = blockIdx.x;
    const uint64_t rm = mb > 0 ? rev_bits(m, mb) : 0;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) {   // r = rev5(b), tx = rev5(a)
        double2 v = x[((uint64_t)r << (t - 5)) + (rm << 5) + tx];
        if (conj_in) v.y = -v.y;
        tile[r][tx] = v;
    }
    __syncthreads();
    for (int a = ty; a < 32; a += 8) {   // output row a, column b = tx
        int rb = (int)rev_bits(tx, 5), ra = (int)rev_bits(a, 5);
        y[((uint64_t)a << (t - 5)) + (m << 5) + tx] = tile[rb][ra];
    }
}

cudaError_t launch_bitrev(const double2 *in, double2 *out, int t, int conj_in, cudaStream_t s) {
    if (t >= 10) {
        uint64_t blocks = 1ull << (t - 10);
        if (blocks > 0x7fffffffull) return cudaErrorInvalidValue;
        bitrev_tiled<<<(unsigned)blocks, 256, 0, s>>>(in, out, t, conj_in);
    } else {
        bitrev_direct<<<1, 256, 0, s>>>(in, out, t, conj_in);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K2: one radix-2 stage
// Fig 3.9: L = 2^q; for col' = 0, L, ...; row < L/2:
//   c = weight(row)*x(col'+row+L/2); d = x(col'+row); x(col'+row) = d + c; x(col'+row+L/2) = d - c
// with weight(row) = omega_L^row = omega_n^(row * n/L) from the two-level table.
__global__ void radix2_stage_kernel(const double2 *__restrict__ in, double2 *__restrict__ out, int t, int q,
                                    const double2 *__restrict__ hi, const double2 *__restrict__ lo, int h,
                                    int conj_out) {
    const uint64_t half = 1ull << (t - 1);
    const int lh = q - 1;   // log2(L/2)
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < half;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t col = g >> lh, row = g & ((1ull << lh) - 1);
        uint64_t lo_i = (col << q) + row, hi_i = lo_i + (1ull << lh);
        uint64_t e = row << (t - q);
        double2 w = cmul(__ldg(hi + (e >> h)), __ldg(lo + (e & ((1ull << h) - 1))));
        double2 c = cmul(w, in[hi_i]);
        double2 dd = in[lo_i];
        double2 a = cadd(dd, c), b = csub(dd, c);
        if (conj_out) {
            a.y = -a.y;
            b.y = -b.y;
        }
        out[lo_i] = a;
        out[hi_i] = b;
    }
}

cudaError_t launch_radix2_stage(const double2 *in, double2 *out, int t, int q, const double2 *tw_hi,
                                const double2 *tw_lo, int hbits, int conj_out, cudaStream_t s) {
    uint64_t half = 1ull << (t - 1);
    uint64_t blocks = (half + 255) / 256;
    if (blocks > (uint64_t)sm_count() * 64) blocks = (uint64_t)sm_count() * 64;
    radix2_stage_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, t, q, tw_hi, tw_lo, hbits, conj_out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K6: cyclic phase
// Rank d received R_d[s][c] = omega_n^(s*k1) A_s[k1] for k1 = d + P*c from every
// source s (Fig 5.9 layout: source s's chunk at offset s*psize/m).
// The paper's stages q = breakpoint..t with weightcyclic (Fig 5.7) are,
// after that twiddle, the P-point DFT  out_d[c + chunk*k2] = sum_s omega_P^(s*k2) R_d[s][c].
template <int P>
__global__ void __launch_bounds__(256) pcombine_kernel(const double2 *__restrict__ recv, double2 *__restrict__ out,
                                                       int64_t chunk, int conj_out) {
    // U columns c per thread, all loads issued before any DFT (memory-level
    // parallelism of a streaming pass: P*U independent 16-byte loads in flight)
    constexpr int U = P >= 8 ? 2 : 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c0 < chunk; c0 += U * stride) {
        double2 v[U][P];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + u * stride;
            if (c < chunk) {
#pragma unroll
                for (int s = 0; s < P; ++s) v[u][s] = __ldg(recv + s * chunk + c);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + u * stride;
            if (c >= chunk) break;
            dft_reg<P>(v[u]);
#pragma unroll
            for (int k = 0; k < P; ++k) {
                double2 o = v[u][k];
                if (conj_out) o.y = -o.y;
                __stcs(out + c + chunk * k, o);
            }
        }
    }
}

cudaError_t launch_pcombine(const double2 *recv, double2 *out, int64_t chunk, int P, int conj_out,
                            cudaStream_t s) {
    // one wave of 8 CTAs of 256 threads per SM, each thread U columns per sweep
    const int sms = sm_count();
    int64_t blocks = (chunk + 255) / 256;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    switch (P) {
    case 2: pcombine_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, conj_out); break;
    case 4: pcombine_kernel<4><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, conj_out); break;
    case 8: pcombine_kernel<8><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, conj_out); break;
    case 16: pcombine_kernel<16><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, conj_out); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// K6' psplit<P>: the low-end breakpoint's phase 1 (Fig 5.7 with breakpoint = log2 m + 1,
// P:665/694).  Rank r holds x[r + P*j'] (its block of P_n x); stages 1..log2 P
// of Fig 3.9 on that block are the P-point DFTs over j' = c + chunk*s (stride psize/m),
// and the weightcyclic factor of the following cyclic phase (Fig 4.4),
// omega_n^((r + P*c)*u), is applied before the element leaves for rank u.
template <int P>
__global__ void __launch_bounds__(256) psplit_kernel(const double2 *__restrict__ in, double2 *__restrict__ send,
                                                     int64_t chunk, uint64_t r, uint64_t nmask,
                                                     const double2 *__restrict__ tw_hi,
                                                     const double2 *__restrict__ tw_lo, int hbits, int conj_in) {
    const uint64_t lomask = (1ull << hbits) - 1;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < chunk;
         c += (int64_t)gridDim.x * blockDim.x) {
        double2 v[P];
#pragma unroll
        for (int s = 0; s < P; ++s) {
            v[s] = __ldg(in + c + chunk * s);
            if (conj_in) v[s].y = -v[s].y;
        }
        dft_reg<P>(v);
        const uint64_t e1 = (r + (uint64_t)P * (uint64_t)c) & nmask;
        __stcs(send + c, v[0]);
#pragma unroll
        for (int u = 1; u < P; ++u) {
            const uint64_t e = (e1 * (uint64_t)u) & nmask;
            const double2 w = cmul(__ldg(tw_hi + (e >> hbits)), __ldg(tw_lo + (e & lomask)));
            __stcs(send + c + chunk * u, cmul(v[u], w));
        }
    }
}

cudaError_t launch_psplit(const double2 *in, double2 *send, int64_t chunk, int P, int64_t r, int64_t n,
                          const double2 *tw_hi, const double2 *tw_lo, int hbits, int conj_in, cudaStream_t s) {
    const int sms = sm_count();
    int64_t blocks = (chunk + 255) / 256;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    const uint64_t nm = (uint64_t)n - 1;
    switch (P) {
    case 2: psplit_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(in, send, chunk, r, nm, tw_hi, tw_lo, hbits, conj_in); break;
    case 4: psplit_kernel<4><<<(unsigned)blocks, 256, 0, s>>>(in, send, chunk, r, nm, tw_hi, tw_lo, hbits, conj_in); break;
    case 8: psplit_kernel<8><<<(unsigned)blocks, 256, 0, s>>>(in, send, chunk, r, nm, tw_hi, tw_lo, hbits, conj_in); break;
    case 16: psplit_kernel<16><<<(unsigned)blocks, 256, 0, s>>>(in, send, chunk, r, nm, tw_hi, tw_lo, hbits, conj_in); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// pcombine with the low-end breakpoint's inner twiddle: block s of recv is the
// (M/P)-point FFT of source s's W[s][c]; column c is scaled by omega_M^(s*c) =
// omega_n^(P*s*c) before the P-point DFT over s (exec.cu's lowend derivation).
template <int P>
__global__ void __launch_bounds__(256) pcombine_tw_kernel(const double2 *__restrict__ recv,
                                                          double2 *__restrict__ out, int64_t chunk, uint64_t nmask,
                                                          const double2 *__restrict__ tw_hi,
                                                          const double2 *__restrict__ tw_lo, int hbits,
                                                          int conj_out) {
    const uint64_t lomask = (1ull << hbits) - 1;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < chunk;
         c += (int64_t)gridDim.x * blockDim.x) {
        double2 v[P];
#pragma unroll
        for (int s = 0; s < P; ++s) v[s] = __ldg(recv + s * chunk + c);
        const uint64_t e1 = ((uint64_t)P * (uint64_t)c) & nmask;
#pragma unroll
        for (int s = 1; s < P; ++s) {
            const uint64_t e = (e1 * (uint64_t)s) & nmask;
            v[s] = cmul(v[s], cmul(__ldg(tw_hi + (e >> hbits)), __ldg(tw_lo + (e & lomask))));
        }
        dft_reg<P>(v);
#pragma unroll
        for (int k = 0; k < P; ++k) {
            double2 o = v[k];
            if (conj_out) o.y = -o.y;
            __stcs(out + c + chunk * k, o);
        }
    }
}

cudaError_t launch_pcombine_tw(const double2 *recv, double2 *out, int64_t chunk, int P, int64_t n,
                               const double2 *tw_hi, const double2 *tw_lo, int hbits, int conj_out, cudaStream_t s) {
    const int sms = sm_count();
    int64_t blocks = (chunk + 255) / 256;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    const uint64_t nm = (uint64_t)n - 1;
    switch (P) {
    case 2: pcombine_tw_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, nm, tw_hi, tw_lo, hbits, conj_out); break;
    case 4: pcombine_tw_kernel<4><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, nm, tw_hi, tw_lo, hbits, conj_out); break;
    case 8: pcombine_tw_kernel<8><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, nm, tw_hi, tw_lo, hbits, conj_out); break;
    case 16: pcombine_tw_kernel<16><<<(unsigned)blocks, 256, 0, s>>>(recv, out, chunk, nm, tw_hi, tw_lo, hbits, conj_out); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// Chunked form (SURVEY §8(e) overlap): chunk g of the receive buffer, [src][count],
// column c_local -> global column c = inner_len*(goff + (o % wg) + f1*(o / wg)) + i.
template <int P>
__global__ void __launch_bounds__(256) pcombine_chunk_kernel(const double2 *__restrict__ recv,
                                                             double2 *__restrict__ out, int64_t count, int li,
                                                             int lwg, int64_t f1, int64_t goff,
                                                             int64_t out_stride, int conj_out) {
    for (int64_t cl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cl < count;
         cl += (int64_t)gridDim.x * blockDim.x) {
        double2 v[P];
#pragma unroll
        for (int s = 0; s < P; ++s) v[s] = __ldg(recv + s * count + cl);
        dft_reg<P>(v);
        const int64_t i = cl & ((1ll << li) - 1), o = cl >> li;
        const int64_t c = ((goff + (o & ((1ll << lwg) - 1)) + f1 * (o >> lwg)) << li) + i;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            double2 w = v[k];
            if (conj_out) w.y = -w.y;
            __stcs(out + c + out_stride * k, w);
        }
    }
}

cudaError_t launch_pcombine_chunk(const double2 *recv, double2 *out, int64_t count, int P, int64_t inner_len,
                                  int64_t wg, int64_t f1, int64_t goff, int64_t out_stride, int conj_out,
                                  cudaStream_t s) {
    int li = 0, lwg = 0;
    while (((int64_t)1 << li) < inner_len) ++li;
    while (((int64_t)1 << lwg) < wg) ++lwg;
    int64_t blocks = (count + 255) / 256;
    if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
    switch (P) {
    case 2: pcombine_chunk_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(recv, out, count, li, lwg, f1, goff, out_stride, conj_out); break;
    case 4: pcombine_chunk_kernel<4><<<(unsigned)blocks, 256, 0, s>>>(recv, out, count, li, lwg, f1, goff, out_stride, conj_out); break;
    case 8: pcombine_chunk_kernel<8><<<(unsigned)blocks, 256, 0, s>>>(recv, out, count, li, lwg, f1, goff, out_stride, conj_out); break;
    case 16: pcombine_chunk_kernel<16><<<(unsigned)blocks, 256, 0, s>>>(recv, out, count, li, lwg, f1, goff, out_stride, conj_out); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ input generator (harness)
__device__ __forceinline__ double splitmix_u(uint64_t seed, uint64_t idx) {
    uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-52 - 1.0;
}

__global__ void gen_uniform_kernel(uint64_t seed, int64_t first, int64_t stride, int64_t count,
                                   double2 *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t g = (uint64_t)first + (uint64_t)stride * (uint64_t)i;
        out[i] = make_double2(splitmix_u(seed, 2 * g), splitmix_u(seed, 2 * g + 1));
    }
}

cudaError_t launch_gen_uniform(uint64_t seed, int64_t first, int64_t stride, int64_t count, double2 *out,
                               cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > (int64_t)sm_count() * 32) blocks = (int64_t)sm_count() * 32;
    gen_uniform_kernel<<<(unsigned)blocks, 256, 0, s>>>(seed, first, stride, count, out);
    return cudaGetLastError();
}

}  // namespace moa
