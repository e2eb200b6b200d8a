// moa_internal.h -- types shared by the host plan code and the CUDA kernels.
// Not part of the public ABI (include/moa_fft.h is).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace moa {

constexpr int FMAX_LOG = 13;            // largest on-chip FFT length per pass: 2^13 points
constexpr int FMAX = 1 << FMAX_LOG;     // (128 KiB of complex128 per CTA)
constexpr int TF_MAX = 8192;            // T*F <= TF_MAX elements per CTA tile

// One lifted pass: for every tile, T independent F-point
// DFTs along an axis of stride in_f (the paper's butterfly stages of one
// lifted level, Fig 3.7 basic block grouped into radix-16 register kernels),
// an optional twiddle multiply omega_n^(alpha + beta*k) (Fig 4.4's weightcyclic
// scaling folded into the lifted form), and a store either in place (middle
// passes) or to the transposed/natural output index K (last pass, the
// reshape-transpose of P:49-53) or the all-to-all send layout (p > 1, Fig 5.9).
struct PassDesc {
    const double2 *src;
    double2 *dst;
    const double2 *tw_hi;   // omega_n^(e << hbits) for the two-level table   (sign -1)
    const double2 *tw_lo;   // omega_n^e, e < 2^hbits                          (sign -1)
    const double2 *tw_f;    // omega_FMAX^e, e < FMAX: intra-pass stage twiddles (sign -1)
    // tile id -> (u, v, w):  u = id % U, v = (id / U) % V, w = id / (U * V)
    int64_t U, V;           // powers of two
    int lU, lV;             // log2 U, log2 V
    // input element (tile, t, f): in_u*u + in_v*v + in_w*w + in_t*t + in_f*f
    int64_t in_u, in_v, in_w, in_t, in_f;
    // last pass: output index K = K_u*u + K_v*v + K_w*w + K_t*t + K_k*k
    int64_t K_u, K_v, K_w, K_t, K_k;
    // output address of point k of transform t: out_u*u + out_v*v + out_w*w + out_t*t + out_k*k
    // (= the input map for in-place middle passes, K for the last pass, K's send slot when packing)
    int64_t out_u, out_v, out_w, out_t, out_k;
    // twiddle exponent e = alpha + beta*k (mod n),
    //   alpha = a_u*u + a_v*v + a_w*w + a_t*t,  beta = b_u*u + b_v*v + b_w*w + b_t*t
    //   (+ the constants a_c, b_c)
    int64_t a_c, a_u, a_v, a_w, a_t;
    int64_t b_c, b_u, b_v, b_w, b_t;
    uint64_t nmask;         // n - 1 (the GLOBAL n of the transform)
    int hbits;              // split of the two-level table
    int tbits;              // log2 n
    int last;               // 1: store to K (or its pack); 0: store in place at (t, k) of the input view
    int twiddle;            // 1: multiply by omega_n^e before the store
    int conj_in, conj_out;  // sign +1 is computed as conj(FFT_-1(conj x))
    int in_tfast, out_tfast;// lane->(t, j) order of the global-facing stages
    int pack_lp;            // >= 0: general send layout addr = (K & (P-1)) * pack_chunk + (K >> pack_lp)
                            //       (only for a single-level local transform; else out_* is affine)
    int64_t pack_chunk;
    int64_t in_shift;       // subtracted from every input address (src is a window of the view)
    int64_t out_shift;      // subtracted from every in-place output address (dst is a window)
    // p > 1 fused exchange (MOA_XCHG_P2P): the element for destination rank dst is
    // stored at peer[dst] + peer_off + slot (peer[] = the destinations' receive buffers,
    // NVLink-mapped; peer_off = this rank's source block); NULL peer[0] = send buffer
    double2 *peer[16];
    int64_t peer_off;
    // batched transforms: tile id = bi * 2^ltiles + tile-in-transform; transform bi is
    // offset by bi * bstride elements in src and dst (bstride 0 = no batch)
    int ltiles;
    int64_t bstride;
    // programmatic dependent launch: the kernel is launched before its predecessor on
    // the stream has finished; it signals its own dependents at once and waits for the
    // predecessor's grid (griddepcontrol.wait) before touching global data
    int pdl;
};

// L2-fused last two passes (persistent kernel): the middle pass of a 3-level
// lifting writes row groups into an L2-resident scratch ring that the last
// pass consumes, so HBM sees the traffic of two passes instead of three.
struct FusedDesc {
    PassDesc p2, p3;             // the middle and the last pass (src/dst windows set per group)
    const int *items;            // schedule: item -> (kind << 30) | (group << 16) | tile
    int64_t total_items;
    unsigned long long *claim;   // work counter
    unsigned long long *done2;   // per group: finished middle-pass tiles
    unsigned long long *done3;   // per group: finished last-pass tiles
    unsigned long long epoch;    // execute index (counters are monotone across executes)
    int tiles2, tiles3;          // tiles per group of each kind
    int groups, slots;
    int64_t rows_per_group_elems;  // elements of one group in the scratch ring
    double2 *scratch;            // slots * rows_per_group_elems
    int64_t f2f3;                // elements per row (F2 * F3)
    int discard;                 // L2 discard of consumed scratch lines
    int ticket;                  // 1: one item per CTA (fused_ticket_kernel); 0: persistent TMA kernel
    const double2 *work;         // middle-pass input (whole view)
    double2 *out;                // last-pass output
};

// host-side launchers (kernels.cu / fft_inst.cu)
int sm_count();   // SM count of the current device (cached per device)
// the persistent TMA-fed 4096-point pass (bigpass.cu): T = 2 tiles, one CTA per SM
int big_supported(int logF, int T);
cudaError_t prepare_big_kernels();
cudaError_t launch_big(const PassDesc &d, const CUtensorMap &map, int64_t tiles, cudaStream_t s);
int pass_supported(int logF, int T);
size_t pass_smem_bytes(int logF, int T);
int pass_threads(int logF, int T);
cudaError_t launch_pass(int logF, int T, const PassDesc &d, int64_t tiles, cudaStream_t s);
// the row pass with its transposed store issued as bulk-tensor stores from shared memory
cudaError_t launch_pass_tmast(int logF, int T, const PassDesc &d, const CUtensorMap &omap, int64_t tiles,
                              cudaStream_t s);
cudaError_t prepare_pass_kernels();    // raise the dynamic smem limits once
// TMA-staged persistent pass (src 1: column tile, 2: row tile); grid 0 = unsupported
int pass_tma_grid(int logF, int T, int src);
cudaError_t launch_pass_tma(int logF, int T, int src, const PassDesc &d, const CUtensorMap &map, int64_t tiles,
                            int grid, cudaStream_t s);
// prefetching persistent pass (fft_pass_pf_kernel); grid 0 = unsupported
int pass_pf_grid(int logF, int T);
cudaError_t launch_pass_pf(int logF, int T, const PassDesc &d, int64_t tiles, int grid, cudaStream_t s);
int fused_supported(int logF2, int T2, int logF3, int T3);
cudaError_t launch_fused(int logF2, int T2, int logF3, int T3, const FusedDesc &fd, const CUtensorMap &m2,
                         const CUtensorMap &m3, int grid, cudaStream_t s);
int fused_grid(int logF2, int T2, int logF3, int T3);

cudaError_t launch_bitrev(const double2 *in, double2 *out, int t, int conj_in, cudaStream_t s);
cudaError_t launch_radix2_stage(const double2 *in, double2 *out, int t, int q,
                                const double2 *tw_hi, const double2 *tw_lo, int hbits,
                                int conj_out, cudaStream_t s);
cudaError_t launch_pcombine(const double2 *recv, double2 *out, int64_t chunk, int P,
                            int conj_out, cudaStream_t s);
// one chunk g of the chunked exchange: recv holds [src][count] (stride count); column
// c_local of the chunk is global column (inner_len)*(goff + (o % wg) + f1*(o / wg)) + i,
// o = c_local / inner_len, i = c_local % inner_len; out[c + out_stride*k2]
cudaError_t launch_pcombine_chunk(const double2 *recv, double2 *out, int64_t count, int P, int64_t inner_len,
                                  int64_t wg, int64_t f1, int64_t goff, int64_t out_stride, int conj_out,
                                  cudaStream_t s);
// low-end breakpoint phase 1 (rank r): Z_c[u] = sum_s x[c + chunk*s] omega_P^(s*u),
// times omega_n^((r + P*c)*u), stored at send[u*chunk + c]
cudaError_t launch_psplit(const double2 *in, double2 *send, int64_t chunk, int P, int64_t r, int64_t n,
                          const double2 *tw_hi, const double2 *tw_lo, int hbits, int conj_in, cudaStream_t s);
// low-end breakpoint phase 3: v[s] = recv[s*chunk + c] * omega_n^(P*s*c), P-point DFT,
// out[c + chunk*k]
cudaError_t launch_pcombine_tw(const double2 *recv, double2 *out, int64_t chunk, int P, int64_t n,
                               const double2 *tw_hi, const double2 *tw_lo, int hbits, int conj_out, cudaStream_t s);
cudaError_t launch_gen_uniform(uint64_t seed, int64_t first, int64_t stride, int64_t count,
                               double2 *out, cudaStream_t s);

}  // namespace moa

// per-length launchers defined by fft_inst.cu compiled with -DMOA_INST_LOGF=<f>
#define MOA_DECLARE_INST(f)                                                                 \
    namespace moa {                                                                         \
    cudaError_t launch_pass_f##f(int T, const PassDesc &d, int64_t tiles, cudaStream_t s);  \
    cudaError_t prepare_pass_f##f();                                                        \
    cudaError_t launch_pass_tma_f##f(int T, int src, const PassDesc &d, const CUtensorMap &map, \
                                     int64_t tiles, int grid, cudaStream_t s);              \
    int grid_pass_tma_f##f(int T, int src);                                                 \
    cudaError_t launch_pass_pf_f##f(int T, const PassDesc &d, int64_t tiles, int grid, cudaStream_t s); \
    int grid_pass_pf_f##f(int T);                                                           \
    cudaError_t launch_pass_tmast_f##f(int T, const PassDesc &d, const CUtensorMap &omap, int64_t tiles, \
                                       cudaStream_t s);                                     \
    }
MOA_DECLARE_INST(1)
MOA_DECLARE_INST(2)
MOA_DECLARE_INST(3)
MOA_DECLARE_INST(4)
MOA_DECLARE_INST(5)
MOA_DECLARE_INST(6)
MOA_DECLARE_INST(7)
MOA_DECLARE_INST(8)
MOA_DECLARE_INST(9)
MOA_DECLARE_INST(10)
MOA_DECLARE_INST(11)
MOA_DECLARE_INST(12)
MOA_DECLARE_INST(13)
