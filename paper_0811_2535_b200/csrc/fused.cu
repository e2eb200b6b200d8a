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

// release-ordered increment: the CTA's prior writes (ordered before this thread
// by the preceding __syncthreads) are visible to any thread that acquires the new value
__device__ __forceinline__ void red_release_add(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
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

// Ticket-kernel wait: poll relaxed, then one acquire once the target is reached (an
// acquire load compiles to an L1 invalidation, CCTL.IVALL; polling with it would
// invalidate L1 on every spin).  The consumer reads the producer's data with
// ld.global.cg (L2) only.
__device__ __forceinline__ void wait_geq_relaxed(const unsigned long long *p, unsigned long long target) {
    if (ld_relaxed_u64(p) < target) {
        unsigned ns = 32;
        while (ld_relaxed_u64(p) < target) {
            __nanosleep(ns);
            if (ns < 512) ns <<= 1;
        }
    }
    (void)ld_acquire_u64(p);
}

template <int F2, int T2, int F3, int T3>
struct FusedShape {
    static constexpr int NT = PassShape<F2, T2>::NT;
    static_assert(PassShape<F3, T3>::NT == NT, "fused passes need equal block sizes");
    using S2 = TmaShape<F2, T2, 1>;
    using S3 = TmaShape<F3, T3, 2>;
    static constexpr size_t BUF = S2::BUF > S3::BUF ? S2::BUF : S3::BUF;
    static constexpr size_t TW = S2::TW > S3::TW ? S2::TW : S3::TW;
    static constexpr size_t SMEM = 128 + 2 * BUF + TW + 64;
    static constexpr int MINB = (T2 * F2 <= 2048) ? 3 : 1;
};

// row tile of the scratch ring: dims {2F3 doubles, T3 rows (stride F2F3), F2 (stride F3), slots}
template <int F3, int T3>
__device__ __forceinline__ void tma_issue_scratch(const CUtensorMap *map, uint64_t *bar, double2 *dst, int tile,
                                                  int slot) {
    using S3 = TmaShape<F3, T3, 2>;
    mbar_expect_tx(bar, S3::BOX_BYTES * S3::NBOX);
#pragma unroll
    for (int k = 0; k < S3::NBOX; ++k) tma_load_4d(dst + k * S3::FB * T3, map, bar, 2 * S3::FB * k, 0, tile, slot);
}

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Persistent, double-buffered: while item i is transformed in buffer i&1 the
// next item has already been claimed and (when its inputs are ready) its tile
// is streaming into the other buffer by TMA -- from HBM for a middle-pass item,
// from the L2-resident scratch ring for a last-pass item.
template <int F2, int T2, int F3, int T3>
__global__ void __launch_bounds__(FusedShape<F2, T2, F3, T3>::NT, FusedShape<F2, T2, F3, T3>::MINB)
    fused_kernel(const FusedDesc fd, const __grid_constant__ CUtensorMap map2, const __grid_constant__ CUtensorMap map3) {
    using SH = FusedShape<F2, T2, F3, T3>;
    extern __shared__ unsigned char smraw[];
    // align by pointer arithmetic (an integer round trip would lose the shared
    // address space and turn every exchange access into a generic LD/ST)
    unsigned char *base = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
    auto buf = [&](int i) { return reinterpret_cast<double2 *>(base + i * SH::BUF); };
    double2 *tw = reinterpret_cast<double2 *>(base + 2 * SH::BUF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(base + 2 * SH::BUF + SH::TW);
    __shared__ long long s_item[2];
    __shared__ int s_issued[2];
    const int tid = threadIdx.x;
    const unsigned long long claim_base = fd.epoch * (unsigned long long)(fd.total_items + gridDim.x);
    const unsigned long long tgt2 = (fd.epoch + 1) * (unsigned long long)fd.tiles2;
    const unsigned long long tgt3 = (fd.epoch + 1) * (unsigned long long)fd.tiles3;

    // thread 0: start the copy of `item` into buffer b (wait for its inputs only if `block`)
    auto try_issue = [&](long long item, int b, bool block) -> bool {
        const int code = __ldg(fd.items + item);
        const int kind = code >> 30, g = (code >> 16) & 0x3fff, tile = code & 0xffff;
        if (kind == 1) {
            if (ld_acquire_u64(fd.done2 + g) < tgt2) {
                if (!block) return false;
                wait_geq(fd.done2 + g, tgt2);
            }
            fence_proxy_async_global();   // the generic-proxy scratch writes are visible to TMA
            fence_proxy_async();
            tma_issue_scratch<F3, T3>(&map3, &bar[b], buf(b), tile, g % fd.slots);
        } else {
            fence_proxy_async();
            tma_issue_tile<F2, T2, 1>(&map2, &bar[b], buf(b), fd.p2, (int64_t)g * fd.tiles2 + tile);
        }
        return true;
    };

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        const long long first = (long long)(atomicAdd(fd.claim, 1ull) - claim_base);
        s_item[0] = first;
        s_issued[0] = 1;
        if (first < fd.total_items) try_issue(first, 0, true);
    }
    unsigned uses[2] = {0, 0};
    for (int it = 0;; ++it) {
        const int b = it & 1;
        __syncthreads();   // previous item finished (buffer b^1, twiddle tables free)
        const long long item = s_item[b];
        if (item >= fd.total_items) break;
        const int code = __ldg(fd.items + item);
        const int kind = code >> 30, g = (code >> 16) & 0x3fff, tile = code & 0xffff;
        if (tid == 0) {
            // claim the next item and prefetch it into the other buffer if its inputs are ready
            const long long nxt = (long long)(atomicAdd(fd.claim, 1ull) - claim_base);
            s_item[b ^ 1] = nxt;
            s_issued[b ^ 1] = (nxt < fd.total_items) ? (int)try_issue(nxt, b ^ 1, false) : 1;
            if (kind == 0 && g >= fd.slots) wait_geq(fd.done3 + (g - fd.slots), tgt3);   // slot free
            if (!s_issued[b]) try_issue(item, b, true);
        }
        __syncthreads();
        mbar_wait(&bar[b], uses[b] & 1);
        uses[b]++;
        const int slot = g % fd.slots;
        double2 *slot_ptr = fd.scratch + (int64_t)slot * fd.rows_per_group_elems;
        const int64_t shift = (int64_t)g * fd.rows_per_group_elems;
        if (kind == 0) {
            TileIO io{fd.work, slot_ptr, 0, shift};
            tile_fft<F2, T2, 1, SyncHook, 0, 0>(buf(b), tw, fd.p2, io, (int64_t)g * fd.tiles2 + tile, buf(b),
                                               SyncHook());
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(fd.done2 + g, 1ull);
            }
        } else {
            if (fd.discard) {
                // the staged scratch lines are dead: drop them from L2 without write-back
                constexpr int LINES_PER_SEG = F3 * 16 / 128;
                for (int i = tid; i < T3 * LINES_PER_SEG; i += SH::NT) {
                    const int t = i / LINES_PER_SEG, l = i % LINES_PER_SEG;
                    const double2 *a = slot_ptr + (int64_t)tile * F3 + (int64_t)t * fd.f2f3 + l * 8;
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
                }
            }
            TileIO io{slot_ptr, fd.out, shift, 0};
            tile_fft<F3, T3, 2, SyncHook, 0, 1>(buf(b), tw, fd.p3, io, (int64_t)g + (int64_t)fd.groups * tile,
                                               buf(b), SyncHook());
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(fd.done3 + g, 1ull);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Ticket variant: one work item per CTA, no TMA, no persistence.  Each CTA
// takes the next ticket from a global counter, so every item with a smaller
// ticket already belongs to a resident CTA: waiting on it cannot deadlock.
// The tile itself is the plain pass tile (register gathers straight from
// global memory), which keeps 4 CTAs per SM resident like fft_pass_kernel.
//   middle-pass item: work (HBM, evict-first) -> scratch slot (L2)
//   last-pass item:   scratch slot (L2, ld.cg) -> out (HBM, streaming store),
//                     then the consumed scratch lines are discarded from L2.
template <int F2, int T2, int F3, int T3>
struct TicketShape {
    static constexpr int NT = PassShape<F2, T2>::NT;
    static_assert(PassShape<F3, T3>::NT == NT, "fused passes need equal block sizes");
    static constexpr size_t SMEM = PassShape<F2, T2>::SMEM > PassShape<F3, T3>::SMEM ? PassShape<F2, T2>::SMEM
                                                                                      : PassShape<F3, T3>::SMEM;
    static constexpr size_t XCH2 = PassShape<F2, T2>::XCH, XCH3 = PassShape<F3, T3>::XCH;
    static constexpr int MINB = PassShape<F2, T2>::MINB < PassShape<F3, T3>::MINB ? PassShape<F2, T2>::MINB
                                                                                  : PassShape<F3, T3>::MINB;
};

template <int F2, int T2, int F3, int T3>
__global__ void __launch_bounds__(TicketShape<F2, T2, F3, T3>::NT, TicketShape<F2, T2, F3, T3>::MINB)
    fused_ticket_kernel(const FusedDesc fd) {
    using SH = TicketShape<F2, T2, F3, T3>;
    extern __shared__ double2 sm[];
    __shared__ int s_code;
    const int tid = threadIdx.x;
    if (tid == 0) {
        // ticket: blockIdx (CTAs are dispatched in index order, so every smaller
        // index is resident or finished) or, with fd.ticket == 2, a global counter
        const unsigned long long ticket =
            fd.ticket == 2 ? atomicAdd(fd.claim, 1ull) - fd.epoch * (unsigned long long)fd.total_items : blockIdx.x;
        const int code = __ldg(fd.items + ticket);
        const int kind = code >> 30, g = (code >> 16) & 0x3fff;
#ifndef MOA_FUSE_NOWAIT   // timing probe only: without the waits the results are wrong
        if (kind == 1) wait_geq_relaxed(fd.done2 + g, (fd.epoch + 1) * (unsigned long long)fd.tiles2);
        else if (g >= fd.slots)
            wait_geq_relaxed(fd.done3 + (g - fd.slots), (fd.epoch + 1) * (unsigned long long)fd.tiles3);
#endif
        s_code = code;
    }
    __syncthreads();
    const int code = s_code;
    const int kind = code >> 30, g = (code >> 16) & 0x3fff, tile = code & 0xffff;
    double2 *slot_ptr = fd.scratch + (int64_t)(g % fd.slots) * fd.rows_per_group_elems;
    const int64_t shift = (int64_t)g * fd.rows_per_group_elems;
    if (kind == 0) {
        TileIO io{fd.work, slot_ptr, 0, shift};
        tile_fft<F2, T2, 0, NoHook, 2, 0, 1>(sm, reinterpret_cast<double2 *>(reinterpret_cast<char *>(sm) + SH::XCH2),
                                          fd.p2, io, (int64_t)g * fd.tiles2 + tile);
    } else {
        TileIO io{slot_ptr, fd.out, shift, 0};
        tile_fft<F3, T3, 0, NoHook, 1, 1, 0>(sm, reinterpret_cast<double2 *>(reinterpret_cast<char *>(sm) + SH::XCH3),
                                          fd.p3, io, (int64_t)g + (int64_t)fd.groups * tile);
        if (fd.discard) {
            __syncthreads();   // every lane has loaded its scratch points
            constexpr int LINES_PER_SEG = F3 * 16 / 128;
            for (int i = tid; i < T3 * LINES_PER_SEG; i += SH::NT) {
                const int t = i / LINES_PER_SEG, l = i % LINES_PER_SEG;
                const double2 *a = slot_ptr + (int64_t)tile * F3 + (int64_t)t * fd.f2f3 + l * 8;
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
            }
        }
    }
    __syncthreads();
    if (tid == 0) red_release_add((kind == 0 ? fd.done2 : fd.done3) + g, 1ull);
}

template <int F2, int T2, int F3, int T3>
static cudaError_t launch_ticket_f(const FusedDesc &fd, cudaStream_t s) {
    using SH = TicketShape<F2, T2, F3, T3>;
    static bool attr = false;
    if (!attr) {
        if (SH::SMEM > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(fused_ticket_kernel<F2, T2, F3, T3>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::SMEM);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    fused_ticket_kernel<F2, T2, F3, T3><<<(unsigned)fd.total_items, SH::NT, SH::SMEM, s>>>(fd);
    return cudaGetLastError();
}

template <int F2, int T2, int F3, int T3>
static cudaError_t launch_f(const FusedDesc &fd, const CUtensorMap &m2, const CUtensorMap &m3, int grid,
                            cudaStream_t s) {
    if (fd.ticket) return launch_ticket_f<F2, T2, F3, T3>(fd, s);
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
    fused_kernel<F2, T2, F3, T3><<<grid, SH::NT, SH::SMEM, s>>>(fd, m2, m3);
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
    X(7, 32, 8, 16)

int fused_supported(int logF2, int T2, int logF3, int T3) {
#define X(a, b, c, d) \
    if (logF2 == a && T2 == b && logF3 == c && T3 == d) return 1;
    MOA_FUSED_LIST(X)
#undef X
    return 0;
}

cudaError_t launch_fused(int logF2, int T2, int logF3, int T3, const FusedDesc &fd, const CUtensorMap &m2,
                         const CUtensorMap &m3, int grid, cudaStream_t s) {
#define X(a, b, c, d) \
    if (logF2 == a && T2 == b && logF3 == c && T3 == d) return launch_f<1 << a, b, 1 << c, d>(fd, m2, m3, grid, s);
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
