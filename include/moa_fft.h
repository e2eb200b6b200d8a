/*
 * moa_fft.h -- C ABI of the B200-native MoA reshape-transpose FFT.
 *
 * The operation (PAPER.md = arXiv 0811.2535, cited P:<line>):
 *   Input x in C^n, n = 2^t, t >= 1; output the FFT of x            (Fig 2.1)
 *   X_k = sum_{j<n} x_j exp(sign * 2*pi*i * j*k / n), no normalisation
 *   computed as the radix-2 Cooley-Tukey FFT of Fig 2.1 / Fig 3.9 (P:103-117,
 *   P:314-333) restructured by dimension lifting ("reshape-transpose"):
 *   local butterfly passes, twiddle scaling, a transpose, more local passes;
 *   and for p > 1 the block/cyclic partition of §4-§5 (Fig 4.9 P:706-747,
 *   Fig 5.7) with the single block->cyclic redistribution of
 *   Fig 5.9 done as an NCCL all-to-all.
 *
 * Data: complex128 = two IEEE doubles (re, im) interleaved, 16-byte aligned,
 * i.e. torch.complex128 / std::complex<double> / double2.
 *
 * Every pointer argument called `in` / `out` in an execute call is a
 * caller-owned DEVICE pointer on the plan's device unless the function name
 * says _host.  The library never frees caller memory.  No function here takes
 * or returns a torch type.  All functions are thread-compatible (one plan per
 * thread at a time); the error message is thread-local.
 *
 * Errors: functions returning int return MOA_OK (0) or a negative MOA_ERR_*
 * code; functions returning a plan return NULL on error.  After any error,
 * moa_fft_last_error() describes it (naming the violated bound for argument
 * errors, as SPEC S:266-274 asks of validate_config).
 */
#ifndef MOA_FFT_H
#define MOA_FFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MOA_OK = 0,
    MOA_ERR_INVALID_N = -1,    /* n is not 2^t with 1 <= t <= 32                       */
    MOA_ERR_INVALID_P = -2,    /* p not a power of two, p != world size, or n/p < p */
    MOA_ERR_INVALID_SIGN = -3, /* sign not -1 or +1                                    */
    MOA_ERR_ALIGN = -4,        /* a device pointer is NULL or not 16-byte aligned        */
    MOA_ERR_NO_DIST = -5,      /* p > 1 (real ranks) without moa_dist_init               */
    MOA_ERR_OOM = -6,          /* device or host allocation failed                     */
    MOA_ERR_CUDA = -7,         /* a CUDA runtime call or kernel launch failed           */
    MOA_ERR_NCCL = -8,         /* libnccl missing or an NCCL call failed                */
    MOA_ERR_INVALID_ARG = -9   /* NULL plan, bad option, or wrong plan kind for the call */
};

typedef struct moa_fft_plan_s *moa_fft_plan_t;

/* Execution modes (moa_fft_options.mode). */
enum {
    MOA_MODE_LIFTED = 0,   /* d(n) lifted passes: the product path  */
    MOA_MODE_LITERAL = 1,  /* the paper's own schedule on the GPU: bit reversal kernel
                              (P_n) + t radix-2 stage kernels (Fig 3.9 butterflies,
                              P:321-327).  Ablation baseline; p == 1 only.               */
    MOA_MODE_EMULATED = 2  /* p > 1 virtual ranks on this one GPU: the same per-rank
                              kernels, the all-to-all done with device copies (tests)    */
};

/* Global transpose (S7, the Fig 5.9 redistribution) for p > 1. */
enum {
    MOA_XCHG_NCCL = 0,     /* last pass packs a send buffer; one NCCL send/recv group   */
    MOA_XCHG_P2P = 1,      /* last pass stores straight into every peer's receive buffer
                              through CUDA-IPC-mapped NVLink pointers (the all-to-all is
                              fused into the butterfly kernel); an 8-byte NCCL all-reduce
                              is the only collective (a barrier).  EMULATED plans: the
                              same stores into the virtual ranks' receive buffers.      */
    MOA_XCHG_P2P_EXTERNAL = 2  /* as P2P, but no NCCL at all: the caller supplies the
                              rank (options.rank), exchanges the IPC handles
                              (moa_fft_ipc_handle / moa_fft_ipc_open) and synchronises
                              all ranks between moa_fft_execute_phase 1 and 2          */
};

typedef struct {
    int mode;            /* MOA_MODE_*                                                */
    int nlift;           /* 0 = default lifting; else number of factors in lift[]      */
    int64_t lift[4];     /* lifting <F1..Fd> (powers of two, product n (p=1) or n/p)   */
    int chunks;          /* p > 1: all-to-all chunks G (0 = default)                   */
    int exchange;        /* MOA_XCHG_* (p > 1)                                         */
    int rank;            /* MOA_XCHG_P2P_EXTERNAL: this process's rank in [0, p)       */
    int64_t batch;       /* p == 1, lifted mode: number of independent length-n
                            transforms stored back to back (transform b at elements
                            [b*n, (b+1)*n) of in and out); 0 or 1 = one transform.
                            Every pass covers the whole batch in one launch.           */
    int breakpoint;      /* p > 1: the stage q at which Fig 5.7's cyclic phase starts
                            (the paper's breakpoint, range [log2 m + 1, log2 psize + 1],
                            P:665).  0 or log2(psize)+1 = the high end: phase 1
                            = the full local psize-point FFT, phase 2 = one m-point DFT
                            (pcombine).  log2(m)+1 = the low end: phase 1 = the
                            m-point DFTs of stages 1..log2 m at local stride psize/m
                            with the weightcyclic factor omega_n^((r+m*c)*u) fused
                            (psplit kernel), then the exchange, then the m FFTs of
                            length psize/m of the received [source][c] blocks (one
                            batched plan; lift[] is ITS lifting, product n/m^2) and an
                            m-point DFT with the factor omega_psize^(s*c) on its loads
                            (pcombine).  Both ends leave X[r + m*i] at out[i] on rank
                            r.  Other values: MOA_ERR_INVALID_ARG (the oracle's Fig 5.7
                            simulation covers every breakpoint).  The low end needs the
                            NCCL exchange (or EMULATED) and psize >= 2m.               */
} moa_fft_options;

typedef struct {
    int64_t n;           /* transform length                                          */
    int t;               /* log2 n                                                    */
    int p;               /* ranks the transform is partitioned over (paper's m)        */
    int rank;            /* this process's rank (0 for p == 1 or emulated)             */
    int sign;            /* -1 forward / +1 the paper's literal EXP(+2 pi i ...)        */
    int mode;            /* MOA_MODE_*                                                */
    int64_t local_n;     /* elements per rank: n / p (the paper's psize)               */
    int passes;          /* kernel passes over the local data (lifting depth d)       */
    int64_t lift[4];     /* lifting factors <F1..Fd>                                  */
    int breakpoint;      /* q at which the cyclic phase starts: log2(psize)+1 (P:289,
                            default) or log2(m)+1 (options.breakpoint)         */
    int chunks;          /* all-to-all chunks G                                       */
    int launches;        /* kernels one execute launches (not counting NCCL's)        */
    int64_t workspace_bytes;  /* device bytes the plan owns                            */
    int64_t hbm_bytes;        /* algorithmic HBM bytes per execute on this rank        */
    int64_t a2a_bytes;        /* bytes this rank sends per execute (p > 1)             */
    int64_t batch;            /* transforms per execute                                */
} moa_fft_info;

/*
 * Create a plan for an n-point transform over p ranks.
 *   n    = 2^t, 1 <= t <= 32 (Fig 2.1 input "n = 2^t, t >= 1"; 2^32 complex128
 *          = 64 GiB per buffer is beyond one 180 GB B200 once in/out/scratch are counted).
 *   p    = 1, or the world size given to moa_dist_init (a power of two, the paper's m)
 *          with n/p >= p (psize >= m).
 *   sign = -1 (forward, conventional) or +1 (the paper's literal EXP(+2*pi*i*row/L)).
 * Binds to the current CUDA device; owns twiddle tables, scratch and (p > 1)
 * send/receive buffers.  For p > 1 the call is collective.  NULL on error.
 */
moa_fft_plan_t moa_fft_plan(int64_t n, int p, int sign);

/*
 * Two-dimensional transform: App. B's Omega applies a 1-D
 * operation to every sub-array along an axis (B.1-B.6), so the 2-D DFT
 *   X[k1][k2] = sum_{j1,j2} x[j1][j2] exp(sign*2*pi*i*(j1*k1/n1 + j2*k2/n2))
 * is the lifted 1-D FFT over the rows followed by the same over the columns.
 *   n1 = 2^t1, 1 <= t1 <= 26 (the column transforms: one pass up to 2^10, else two
 *   lifted passes), n2 = 2^t2 with t2 >= 1 (the rows: a batched lifted 1-D plan),
 *   n1 * n2 <= 2^32.
 * x, X: n1 x n2 complex128, row-major (element (j1, j2) at j1*n2 + j2).  Execute
 * with moa_fft_execute; in == out allowed.  NULL on error (moa_fft_last_error).
 */
moa_fft_plan_t moa_fft_plan_2d(int64_t n1, int64_t n2, int sign);

/*
 * r-dimensional transform, r = 2 or 3, of a row-major shape[0] x ... x shape[r-1]
 * complex128 array: X[k] = sum_j x[j] exp(sign*2*pi*i * sum_a j_a*k_a/shape[a]).
 * The last axis is any power of two (a batched lifted 1-D plan); every other axis is
 * 2^t with 1 <= t <= 26: one pass of DFTs along that strided axis, in place, for
 * t <= 10, else two lifted passes through a plan-owned work buffer (twiddle
 * omega_N^(j2*k1) between them, transposed store); last-but-one axis first.  The
 * product of the extents is <= 2^32.  Execute
 * with moa_fft_execute; in == out allowed.  NULL on error.  (moa_fft_plan_2d is the
 * rank-2 case.)
 */
moa_fft_plan_t moa_fft_plan_nd(int rank, const int64_t *shape, int sign);

/* As moa_fft_plan with explicit options (NULL = defaults).  A lifting whose
 * product is wrong or with a factor outside [2, 8192] is MOA_ERR_INVALID_ARG. */
moa_fft_plan_t moa_fft_plan_ex(int64_t n, int p, int sign, const moa_fft_options *opts);

/*
 * Execute the transform, asynchronously on the plan's stream.
 *   p == 1: in/out hold batch*n elements (batch transforms back to back, natural
 *           order); in == out allowed; in is not modified when in != out.
 *   p > 1 : in/out hold n/p elements of THIS rank in the cyclic layout
 *           in[j] = x[rank + p*j], out[i] = X[rank + p*i] (the paper's xcyclic,
 *           P:799).  Collective: every rank calls it in the same order.
 *   EMULATED plans: in/out hold all p ranks' slices back to back (p*(n/p)).
 * Single-GPU multi-pass plans replay their kernel launches as one CUDA graph per
 * (in, out) pair: the first execute with a new pair captures it (on a private
 * stream) and launches it; the graph only remembers the pointer values, so the
 * caller may free or reuse the buffers afterwards.  (Tuning knobs: every MOA_FFT_*
 * environment variable -- e.g. MOA_FFT_GRAPH=0 -- is ignored unless MOA_FFT_ABLATION=1.)
 * in and out are either the same pointer or disjoint ranges (a partial overlap is
 * MOA_ERR_INVALID_ARG).
 * Returns MOA_OK or MOA_ERR_ALIGN / MOA_ERR_INVALID_ARG / MOA_ERR_CUDA / MOA_ERR_NCCL.
 */
int moa_fft_execute(moa_fft_plan_t plan, const void *in, void *out);

/*
 * End-to-end form: in/out are HOST pointers (pinned for full speed).  Copies
 * in -> device, executes, copies the result back, and synchronises the plan
 * stream before returning.  Same layouts as moa_fft_execute.
 */
int moa_fft_execute_host(moa_fft_plan_t plan, const void *host_in, void *host_out);

/*
 * Pipelined end-to-end form for a stream of `count` independent transforms:
 * host_in[i] -> host_out[i] (HOST pointers, pinned for full speed, same layout
 * as moa_fft_execute_host).  Two device staging pairs and two copy streams let
 * the host->device copy of transform i+1 and the device->host copy of
 * transform i-1 overlap the execute of transform i (PCIe is full duplex).
 * Synchronises before returning; every host_out[i] is then complete.
 * Returns MOA_OK, MOA_ERR_INVALID_ARG (NULL plan, count < 0), MOA_ERR_ALIGN (a
 * NULL buffer), MOA_ERR_OOM, or the first execute / CUDA error.
 */
int moa_fft_execute_host_batch(moa_fft_plan_t plan, int count, const void *const *host_in,
                               void *const *host_out);

/* Free everything the plan owns (synchronises its stream first).  NULL-safe. */
void moa_fft_destroy(moa_fft_plan_t plan);

/* Order the plan's work on `stream` (a cudaStream_t; NULL = legacy default stream). */
int moa_fft_set_stream(moa_fft_plan_t plan, void *stream);

/* Fill *out with the plan's shape, lifting and byte counts. */
int moa_fft_plan_info(moa_fft_plan_t plan, moa_fft_info *out);

/*
 * Per-kernel timing for benchmarks.  While enabled, every kernel an execute
 * launches is bracketed by a CUDA event pair on the plan's stream.
 * moa_fft_get_profile synchronises the stream, aggregates the elapsed times per
 * kernel slot since the last call (then resets), and returns the number of
 * slots written (<= max_stats), or a negative error code.
 */
typedef struct {
    char name[64];              /* e.g. "pass1 fft_pass<F=4096,T=2>", "pcombine<P=8>"     */
    int launches;               /* launches aggregated into this slot                      */
    double total_ms;            /* summed event-measured duration                          */
    int64_t alg_bytes;          /* algorithmic HBM bytes per launch (read + write)         */
} moa_fft_kernel_stat;

int moa_fft_set_profiling(moa_fft_plan_t plan, int enable);
int moa_fft_get_profile(moa_fft_plan_t plan, moa_fft_kernel_stat *stats, int max_stats);

/*
 * Host-only introspection of the plan builder (no GPU needed): the index maps
 * pass `pass` of the lifted local transform uses on rank `rank` of p.
 * For every element the pass touches, enumerated tile by tile, row t by row,
 * point f (so consecutive groups of `F` entries are one F-point transform,
 * F = lifting factor of that pass):
 *   in_idx[i]  = local input index read for point f,
 *   out_idx[i] = index written for output k = f (local work index for middle
 *                passes, natural local output index for the last pass when
 *                p == 1, send-buffer index when p > 1),
 *   tw_exp[i]  = e such that the output is multiplied by exp(-2 pi i e / n)
 *                (-1 when the pass applies no twiddle).
 * Arrays hold n/p entries each (caller-owned host memory).  *F_out receives F.
 * Returns MOA_OK or an error code (same validation as moa_fft_plan_ex).
 */
int moa_fft_describe_pass(int64_t n, int p, int rank, const moa_fft_options *opts, int pass,
                          int64_t *in_idx, int64_t *out_idx, int64_t *tw_exp, int64_t *F_out);

/*
 * Peer-to-peer exchange setup (MOA_XCHG_P2P / MOA_XCHG_P2P_EXTERNAL plans).
 *   moa_fft_ipc_handle: write the 64-byte cudaIpcMemHandle of this rank's receive
 *       buffers (plan-owned, 2 x n/p elements: double-buffered across executes) to
 *       handle_out.
 *   moa_fft_ipc_open: handles = p consecutive 64-byte handles in rank order (this
 *       rank's own entry is ignored); maps every peer's receive buffers into this
 *       process (cudaIpcOpenMemHandle, peer access enabled lazily).  Unmapped by
 *       moa_fft_destroy.
 *   moa_fft_enable_p2p: both steps at once, the handles all-gathered over the
 *       library's NCCL communicator (collective; MOA_XCHG_P2P plans).
 * Errors: MOA_ERR_INVALID_ARG (not a P2P plan, NULL buffer), MOA_ERR_CUDA (IPC),
 * MOA_ERR_NO_DIST / MOA_ERR_NCCL (enable_p2p without or with a failing communicator).
 */
int moa_fft_ipc_handle(moa_fft_plan_t plan, void *handle_out_64B);
int moa_fft_ipc_open(moa_fft_plan_t plan, const void *handles_p_x_64B);
int moa_fft_enable_p2p(moa_fft_plan_t plan);

/*
 * Split execute of a P2P plan, for callers that synchronise the ranks
 * themselves (MOA_XCHG_P2P_EXTERNAL):
 *   phase 1: S5 local lifted passes of `in`; the last pass scales by
 *            omega_n^(rank*K) (S6) and stores every element into its destination
 *            rank's receive buffer (S7, fused).  `out` is ignored.
 *   phase 2: S8 P-point combine of this rank's receive buffer into `out`.
 * Between its phase 1 and phase 2 every rank must wait until all ranks' phase 1
 * work has completed (e.g. cudaStreamSynchronize + a host barrier).  Calls
 * alternate 1, 2, 1, 2, ...; the receive buffers alternate per pair, so one
 * barrier per execute suffices.  moa_fft_execute on a MOA_XCHG_P2P plan is
 * phase 1 + an NCCL barrier + phase 2.  Returns MOA_OK, MOA_ERR_INVALID_ARG
 * (wrong plan kind, handles not opened, phase not 1 or 2), MOA_ERR_ALIGN,
 * MOA_ERR_CUDA.
 */
int moa_fft_execute_phase(moa_fft_plan_t plan, const void *in, void *out, int phase);

/*
 * Host-only (no GPU needed): the default lifting <F1..Fd> the plan builder chooses
 * for an n-point transform over p ranks (of the local length n/p).  lift_out has
 * room for 4 factors; *d_out receives d.  Returns MOA_OK or MOA_ERR_INVALID_N /
 * MOA_ERR_INVALID_P (same bounds as moa_fft_plan) / MOA_ERR_INVALID_ARG (NULL).
 */
int moa_fft_default_lifting(int64_t n, int p, int64_t *lift_out, int *d_out);

/* Thread-local description of the last error ("" if none), naming the violated bound
 * for argument errors. */
const char *moa_fft_last_error(void);

/* Thread-local MOA_ERR_* code of the last error (MOA_OK if none): the code that
 * accompanies moa_fft_last_error()'s message, also for calls that return a plan
 * (NULL) rather than a code.  E.g. moa_fft_plan(6, 1, -1) -> NULL and
 * moa_fft_last_error_code() == MOA_ERR_INVALID_N. */
int moa_fft_last_error_code(void);

/*
 * Distributed setup: one library-owned NCCL communicator per process, created
 * with ncclCommInitRank from a 128-byte ncclUniqueId that rank 0 obtained with
 * moa_dist_unique_id and broadcast (the Python side uses torch.distributed).
 * libnccl.so.2 is resolved at run time (the copy already loaded in the process,
 * else the path in $MOA_NCCL_LIB, else the loader's search path).
 */
int moa_dist_unique_id(void *id_out_128B);
int moa_dist_init(int rank, int p, const void *id_128B);
int moa_dist_finalize(void);

/*
 * Redistributions between the paper's layouts of a distributed n-vector (SURVEY §8(f)
 * N2; Figs 5.2-5.5, 5.8, 5.9).  psize = n/p.
 *   MOA_LAYOUT_BLOCK   rank r holds x[r*psize + i], i < psize             (xblock)
 *   MOA_LAYOUT_CYCLIC  rank r holds x[r + p*j],     j < psize             (xcyclic, P:799,
 *                      the transform's own in/out layout for p > 1)
 *   MOA_LAYOUT_CENTRAL rank 0 holds all n elements in natural order, the other ranks
 *                      none (the paper's processor 0)
 *   route MOA_ROUTE_DIRECT:  one point-to-point round in which every rank sends each
 *                      other rank its part directly (Fig 5.3 / Fig 5.9, P:828-842,
 *                      m(m-1) messages of psize/m for block <-> cyclic,
 *                      P:1043); CENTRAL <-> anything is a scatter / gather (m-1 messages)
 *   route MOA_ROUTE_CENTRAL: block <-> cyclic through processor 0 (Fig 5.4, P:844,
 *                      P:848-874): gather, then scatter -- 2(m-1) messages, every
 *                      element moved twice, processor 0's links the bottleneck
 * The local permutations (the pack of the strided SEND sections and the unpack of the
 * received ones) are CUDA kernels; the transfers are NCCL send/recv groups over the
 * library's communicator (moa_dist_init; collective: every rank calls execute in the
 * same order), or device copies when mode == MOA_MODE_EMULATED (all p ranks' buffers
 * back to back on this GPU: BLOCK / CYCLIC buffers hold p*psize elements, rank r's at
 * offset r*psize; CENTRAL buffers hold n elements) or p == 1.
 *   moa_redist_plan: n = 2^t (1 <= t <= 32), p a power of two <= 16 with psize >= p,
 *     from/to MOA_LAYOUT_*, route MOA_ROUTE_*, mode MOA_MODE_LIFTED (real ranks) or
 *     MOA_MODE_EMULATED.  Owns its scratch (psize elements per rank for the direct block
 *     <-> cyclic routes, n on rank 0 for the central ones).  NULL on error.
 *   moa_redist_execute: in / out device pointers in the layouts above, out of place
 *     (in != out); a rank that holds no elements of a layout may pass NULL for it.
 *     Asynchronous on the plan's stream.  MOA_OK / MOA_ERR_ALIGN / MOA_ERR_INVALID_ARG /
 *     MOA_ERR_CUDA / MOA_ERR_NCCL.
 *   moa_redist_info: messages between distinct ranks per execute (whole job), the largest
 *     number of bytes any one rank sends, and this rank's element counts in and out.
 */
enum { MOA_LAYOUT_BLOCK = 0, MOA_LAYOUT_CYCLIC = 1, MOA_LAYOUT_CENTRAL = 2 };
enum { MOA_ROUTE_DIRECT = 0, MOA_ROUTE_CENTRAL = 1 };
typedef struct moa_redist_s *moa_redist_t;
moa_redist_t moa_redist_plan(int64_t n, int p, int from, int to, int route, int mode);
int moa_redist_execute(moa_redist_t plan, const void *in, void *out);
int moa_redist_set_stream(moa_redist_t plan, void *stream);
int moa_redist_info(moa_redist_t plan, int64_t *messages, int64_t *max_rank_bytes, int64_t *elems_in,
                    int64_t *elems_out);
void moa_redist_destroy(moa_redist_t plan);

/*
 * Test/bench helper (not part of the transform): fill `count` complex128 values
 * at device pointer out with x_g = u(seed, 2g) + i*u(seed, 2g+1),
 * g = first + stride*i, u = SplitMix64 mapped to [-1, 1) (the recipe of
 * moa_inputs.py; bit-identical to it).  stream may be NULL.
 */
int moa_gen_uniform(uint64_t seed, int64_t first, int64_t stride, int64_t count,
                    void *out, void *stream);

/* Library version string. */
const char *moa_fft_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOA_FFT_H */
