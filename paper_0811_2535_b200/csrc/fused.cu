// fused.cu -- the last two lifted passes as one persistent kernel with an
// L2-resident scratch ring (SURVEY §8(a) S3 + S4).
//
// With a 3-level lifting <F1, F2, F3> the middle pass (F2-point transforms
// along the stride-F3 axis of every length-F2*F3 row, twiddle omega_{F2F3})
// and the last pass (F3-point transforms of contiguous segments, transposed
// store) are the paper's "reshape-transpose" applied twice to one row
// ("not necessary blocked in squares ... any number of levels").
// A last-pass tile needs T3 rows (consecutive k1, for contiguous output
// runs), so rows are processed in groups of T3: the middle pass writes a
// group into a scratch slot small enough to stay in the 126 MB L2, the last
// pass reads it back from L2.  HBM then carries one read (middle pass) and one
// write (last pass) of the data: two passes' worth of traffic for three
// passes of butterflies.
//
// Scheduling: a persistent grid claims work items in a host-built order
// (P2(0), P2(1), P3(0), P2(2), P3(1), ...).  An item only waits on items
// claimed before it (P3(g) on all of P2(g); P2(g) on P3(g - slots) to reuse
// the slot), so the earliest unfinished item can always run: no deadlock
// whatever the residency.  Counters are monotone across executes (epoch).
#include "fft_pass.cuh"

namespace moa {

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void wait_geq(const unsigned long long *p, unsigned long long target) {
    if (ld_acquire_u64(p) >= target) return;
    unsigned ns = 32;
    while (ld_acquire_u64(p) < target) {
        __nanosleep(ns);
        if (ns < 512) ns <<= 1;
    }
}

template <int F2, int T2, int F3, int T3>
struct FusedShape {
    static constexpr int NT = PassShape<F2, T2>::NT;
    static_assert(PassShape<F3, T3>::NT == NT, "fused passes need equal block sizes");
    static constexpr size_t SMEM =
        PassShape<F2, T2>::SMEM > PassShape<F3, T3>::SMEM ? PassShape<F2, T2>::SMEM : PassShape<F3, T3>::SMEM;
    static constexpr int MINB = PassShape<F2, T2>::MINB;
};

template <int F2, int T2, int F3, int T3>
__global__ void __launch_bounds__(FusedShape<F2, T2, F3, T3>::NT, FusedShape<F2, T2, F3, T3>::MINB)
    fused_kernel(const FusedDesc fd) {
    extern __shared__ double2 sm[];
    __shared__ long long s_item;
    const unsigned long long claim_base = fd.epoch * (unsigned long long)(fd.total_items + gridDim.x);
    const unsigned long long tgt2 = (fd.epoch + 1) * (unsigned long long)fd.tiles2;
    const unsigned long long tgt3 = (fd.epoch + 1) * (unsigned long long)fd.tiles3;
    for (;;) {
        __syncthreads();   // the previous tile's shared-memory reads are done
        if (threadIdx.x == 0) s_item = (long long)(atomicAdd(fd.claim, 1ull) - claim_base);
        __syncthreads();
        const long long item = s_item;
        if (item >= fd.total_items) break;
        const int code = __ldg(fd.items + item);
        const int kind = code >> 30, g = (code >> 16) & 0x3fff, tile = code & 0xffff;
        const int slot = g % fd.slots;
        double2 *slot_ptr = fd.scratch + (int64_t)slot * fd.rows_per_group_elems;
        const int64_t shift = (int64_t)g * fd.rows_per_group_elems;
        if (kind == 0) {
            if (g >= fd.slots) {
                if (threadIdx.x == 0) wait_geq(fd.done3 + (g - fd.slots), tgt3);
                __syncthreads();
            }
            TileIO io{fd.work, slot_ptr, 0, shift};
            tile_fft<F2, T2, 0, NoHook, 0, 0>(sm, fd.p2, io, (int64_t)g * fd.tiles2 + tile);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(fd.done2 + g, 1ull);
            }
        } else {
            if (threadIdx.x == 0) wait_geq(fd.done2 + g, tgt2);
            __syncthreads();
            TileIO io{slot_ptr, fd.out, shift, 0};
            tile_fft<F3, T3, 0, NoHook, 1, 1>(sm, fd.p3, io, (int64_t)g + (int64_t)(fd.groups) * tile);
            __syncthreads();
            if (fd.discard) {
                // the consumed scratch lines are dead: drop them from L2 without write-back.
                // This tile read T3 segments of F3 elements at slot offsets tile*F3 + t*F2*F3.
                constexpr int LINES_PER_SEG = F3 * 16 / 128;
                for (int i = threadIdx.x; i < T3 * LINES_PER_SEG; i += blockDim.x) {
                    int t = i / LINES_PER_SEG, l = i % LINES_PER_SEG;
                    const double2 *a = slot_ptr + (int64_t)tile * F3 + (int64_t)t * fd.f2f3 + l * 8;
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(fd.done3 + g, 1ull);
            }
        }
    }
}

template <int F2, int T2, int F3, int T3>
static cudaError_t launch_f(const FusedDesc &fd, int grid, cudaStream_t s) {
    using SH = FusedShape<F2, T2, F3, T3>;
    static bool attr = false;
    if (!attr) {
        if (SH::SMEM > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(fused_kernel<F2, T2, F3, T3>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::SMEM);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    fused_kernel<F2, T2, F3, T3><<<grid, SH::NT, SH::SMEM, s>>>(fd);
    return cudaGetLastError();
}

template <int F2, int T2, int F3, int T3>
static int grid_f() {
    using SH = FusedShape<F2, T2, F3, T3>;
    static int cached = 0;
    if (cached) return cached;
    if (SH::SMEM > 48 * 1024)
        cudaFuncSetAttribute(fused_kernel<F2, T2, F3, T3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SH::SMEM);
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<F2, T2, F3, T3>, SH::NT, SH::SMEM);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached = per_sm * sms;
    return cached;
}

// the instantiated (F2, T2, F3, T3) combinations (equal block sizes)
#define MOA_FUSED_LIST(X) \
    X(8, 16, 8, 16)       \
    X(8, 8, 8, 8)         \
    X(9, 8, 9, 8)         \
    X(9, 4, 9, 4)         \
    X(7, 16, 7, 16)       \
    X(8, 16, 9, 8)        \
    X(9, 8, 8, 16)        \
    X(10, 4, 10, 4)       \
    X(10, 8, 10, 8)       \
    X(7, 32, 8, 16)

int fused_supported(int logF2, int T2, int logF3, int T3) {
#define X(a, b, c, d) \
    if (logF2 == a && T2 == b && logF3 == c && T3 == d) return 1;
    MOA_FUSED_LIST(X)
#undef X
    return 0;
}

cudaError_t launch_fused(int logF2, int T2, int logF3, int T3, const FusedDesc &fd, int grid, cudaStream_t s) {
#define X(a, b, c, d) \
    if (logF2 == a && T2 == b && logF3 == c && T3 == d) return launch_f<1 << a, b, 1 << c, d>(fd, grid, s);
    MOA_FUSED_LIST(X)
#undef X
    return cudaErrorInvalidValue;
}

int fused_grid(int logF2, int T2, int logF3, int T3) {
#define X(a, b, c, d) \
    if (logF2 == a && T2 == b && logF3 == c && T3 == d) return grid_f<1 << a, b, 1 << c, d>();
    MOA_FUSED_LIST(X)
#undef X
    return 0;
}

}  // namespace moa
