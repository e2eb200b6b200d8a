// plan_internal.h -- the plan object and the helpers shared by the plan builder
// (plan.cu), the executor (exec.cu) and the C ABI (abi.cu).  Not part of the public
// interface (include/moa_fft.h is).
#pragma once
#include <stdlib.h>

#include <string>
#include <vector>

#include "../../include/moa_fft.h"
#include "moa_internal.h"

namespace moa {

// ------------------------------------------------------------------ errors (plan.cu)
int fail(int code, const char *fmt, ...);
void clear_error();
const char *last_error();
int last_error_code();

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
int dist_sendrecv(const double2 *const *send, const int64_t *send_n, double2 *const *recv, const int64_t *recv_n,
                  int p, int rank, cudaStream_t s, std::string *err);
int dist_allgather_sync(const void *send_dev, void *recv_dev, size_t bytes, cudaStream_t s, std::string *err);

// ------------------------------------------------------------------ small helpers
inline int ilog2(int64_t v) {
    int r = 0;
    while (((int64_t)1 << r) < v) ++r;
    return r;
}
inline bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
// Plan-time tuning knobs (MOA_FFT_*) for ablations and tuning sweeps.  They are read
// ONLY when MOA_FFT_ABLATION=1 is set, so a stray environment variable cannot change
// the product kernels or tile shapes; otherwise every knob takes its default.
inline bool ablation_enabled() {
    const char *s = getenv("MOA_FFT_ABLATION");
    return s && *s && atoi(s) != 0;
}
inline int env_int(const char *name, int dflt) {
    if (!ablation_enabled()) return dflt;
    const char *s = getenv(name);
    return (s && *s) ? atoi(s) : dflt;
}

// ------------------------------------------------------------------ one lifted pass
struct PassPlan {
    int logF, T;
    int64_t tiles;
    PassDesc d;  // src/dst patched at execute
    // TMA-staged persistent variant (0 = plain kernel, 1 = column tile, 2 = row tile)
    int tma = 0;
    int tma_grid = 0;
    int pf_grid = 0;   // > 0: prefetching persistent kernel (fft_pass_pf_kernel)
    int tmast = 0;     // last pass stores through the TMA engine (launch_pass_tmast)
    int big = 0;       // 4096-point pass as the persistent TMA-fed kernel (bigpass.cu)
    CUtensorMap omap;  // its output map (encoded for omap_base)
    const void *omap_base = nullptr;
    int io = 0;        // r-D axis passes: 0 = out -> out (in place), 1 = out -> work, 2 = work -> out
    CUtensorMap map;
    const void *map_base = nullptr;
};

double2 host_root(uint64_t e, uint64_t N);
int encode_pass_map(PassPlan &pp, const void *base);
void choose_tma(PassPlan &pp);

}  // namespace moa

struct moa_fft_plan_s {
    int64_t n = 0, M = 0;
    int64_t batch = 1;   // independent transforms per execute (p == 1)
    // 2-D plans (moa_fft_plan_2d): rows = batched 1-D plan of length n2, col = one pass
    // of n1-point DFTs along the stride-n2 axis, in place on the output
    int64_t n1 = 0, n2 = 0;
    moa_fft_plan_s *rows = nullptr;
    // low-end breakpoint: the P transforms of length n/p^2 each rank runs on its received
    // [source][c] blocks (a batched p = 1 plan)
    moa_fft_plan_s *lowsub = nullptr;
    int t = 0, p = 1, rank = 0, sign = -1, mode = MOA_MODE_LIFTED;
    int d = 0;
    int64_t lift[4] = {0, 0, 0, 0};
    int chunks = 1;
    // chunked NCCL exchange (p > 1, 3-level liftings): the last pass split into G groups
    // of the middle digit; per group: pass -> all-to-all (comm stream) -> combine (side stream)
    std::vector<moa::PassPlan> chunk_last;                   // real ranks: G group passes
    std::vector<std::vector<moa::PassPlan>> rank_chunk_last; // emulated: per virtual rank
    cudaStream_t comm_stream = nullptr, comb_stream = nullptr;
    std::vector<cudaEvent_t> ev_pass, ev_a2a;
    cudaEvent_t ev_comb = nullptr;
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
    std::vector<moa::PassPlan> passes;   // p == 1: all passes; p > 1: phase 1 for rank `rank`; 2-D: the column pass
    std::vector<std::vector<moa::PassPlan>> rank_passes;  // emulated: phase 1 per virtual rank
    int64_t workspace_bytes = 0;
    // L2-fused last two passes (fused.cu)
    bool fused = false;
    moa::FusedDesc fd;
    CUtensorMap fmap2, fmap3;
    int fgrid = 0;
    int *items = nullptr;
    unsigned long long *counters = nullptr;
    double2 *scratch = nullptr;
    unsigned long long epoch = 0;
    // CUDA-graph replay of execute (single-GPU plans): the launches of one execute for
    // the last (in, out) pair, captured on a private stream, replayed with one
    // cudaGraphLaunch on the plan stream
    bool graph_ok = false;
    // low-end breakpoint (options.breakpoint = log2 p + 1): psplit + exchange + local FFT
    bool lowend = false;
    cudaStream_t graph_stream = nullptr;
    cudaGraphExec_t gexec = nullptr;
    const void *g_in = nullptr;
    void *g_out = nullptr;
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

// builder (plan.cu)
int default_lifting(int tl, int64_t *lift, int p);
int choose_T(int logF, int64_t avail);
int build_passes(const moa_fft_plan_s *pl, int rank, int P, std::vector<PassPlan> &out);
// options.breakpoint -> pl->lowend (validation)
int resolve_breakpoint(moa_fft_plan_s *pl, const moa_fft_options *opt);
int build_chunked_last(const moa_fft_plan_s *pl, const PassPlan &last, int G, std::vector<PassPlan> &out);
void free_plan(moa_fft_plan_s *pl);
int setup_fused(moa_fft_plan_s *pl, int kind);
int resolve_lifting(moa_fft_plan_s *pl, const moa_fft_options *opt);
int encode_out_map(PassPlan &pp, const void *base);
int make_plan(int64_t n, int p, int sign, const moa_fft_options *opt, moa_fft_plan_s **res);
int make_plan_nd(int rank, const int64_t *shape, int sign, moa_fft_plan_s **res);

// executor (exec.cu)
bool aligned16(const void *ptr);
int launch_pp(moa_fft_plan_s *pl, PassPlan &pp, int idx, const double2 *src, double2 *dst,
              double2 *const *peers = nullptr, int64_t peer_off = 0);
int run_passes(moa_fft_plan_s *pl, std::vector<PassPlan> &ps, const double2 *in, double2 *out,
               double2 *const *peers = nullptr, int64_t peer_off = 0);
int p2p_phase(moa_fft_plan_s *pl, const double2 *in, double2 *out, int phase);
int execute(moa_fft_plan_s *pl, const double2 *in, double2 *out);
int execute_graph(moa_fft_plan_s *pl, const double2 *in, double2 *out);

}  // namespace moa
