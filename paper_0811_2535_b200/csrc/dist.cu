// dist.cu -- the global transpose: the paper's
// DISTRIBUTE_BLOCK_PARTITIONED_TO_CYCLIC_PARTITIONED of Fig 5.9,
//     xcyclic(myid*psize/m : ...) = xblock(myid : psize-1 : m)          (self copy)
//     SEND(xblock(otherp : psize-1 : m), psize/m, otherp)               (m(m-1) messages)
//     RECEIVE(xcyclic(otherp*psize/m), psize/m, otherp)
// on B200 as one NCCL group of ncclSend/ncclRecv over NVLink/NVSwitch.  The
// strided SEND section is already contiguous: the pass epilogue packed it.
//
// libnccl.so.2 is resolved at run time so the library uses the same NCCL the
// process (torch) already loaded: RTLD_NOLOAD first, then $MOA_NCCL_LIB, then
// the loader search path.
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>

#include <string>

#include "../../include/moa_fft.h"
#include "moa_internal.h"

namespace {

typedef struct ncclComm *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat64 = 8;

struct NcclApi {
    void *handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
ncclComm_t g_comm = nullptr;
double *g_barrier_buf = nullptr;   // 8-byte device word the barrier all-reduces
int g_rank = -1, g_size = 0;

int load_nccl(std::string *err) {
    if (g_nccl.handle) return MOA_OK;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
        const char *p = getenv("MOA_NCCL_LIB");
        if (p && *p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        *err = std::string("cannot load libnccl.so.2: ") + dlerror();
        return MOA_ERR_NCCL;
    }
#define SYM(field, name)                                                   \
    *(void **)&g_nccl.field = dlsym(h, name);                              \
    if (!g_nccl.field) {                                                   \
        *err = std::string("libnccl.so.2 lacks ") + name;                  \
        return MOA_ERR_NCCL;                                               \
    }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
#undef SYM
    g_nccl.handle = h;
    return MOA_OK;
}

std::string nccl_msg(const char *what, ncclResult_t r) {
    return std::string(what) + " failed: " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
}

}  // namespace

namespace moa {

int fail(int code, const char *fmt, ...);

int dist_world(int *rank, int *size) {
    *rank = g_rank;
    *size = g_comm ? g_size : 0;
    return MOA_OK;
}

// S7: recv[s*chunk .. ] <- rank s's send[rank*chunk ..] for every s (Fig 5.9)
int dist_alltoall(const double2 *send, double2 *recv, int64_t chunk, int p, int rank, cudaStream_t s,
                  std::string *err) {
    if (!g_comm) {
        *err = "no communicator (moa_dist_init)";
        return MOA_ERR_NO_DIST;
    }
    cudaError_t ce = cudaMemcpyAsync(recv + rank * chunk, send + rank * chunk, chunk * sizeof(double2),
                                     cudaMemcpyDeviceToDevice, s);
    if (ce != cudaSuccess) {
        *err = std::string("self copy failed: ") + cudaGetErrorString(ce);
        return MOA_ERR_CUDA;
    }
    ncclResult_t r = g_nccl.GroupStart();
    if (r) {
        *err = nccl_msg("ncclGroupStart", r);
        return MOA_ERR_NCCL;
    }
    for (int o = 1; o < p; ++o) {   // otherp != myid, visited in rotated order
        int peer = (rank + o) % p;
        int from = (rank - o + p) % p;
        r = g_nccl.Send(send + peer * chunk, (size_t)chunk * 2, kNcclFloat64, peer, g_comm, s);
        if (!r) r = g_nccl.Recv(recv + from * chunk, (size_t)chunk * 2, kNcclFloat64, from, g_comm, s);
        if (r) {
            g_nccl.GroupEnd();
            *err = nccl_msg("ncclSend/ncclRecv", r);
            return MOA_ERR_NCCL;
        }
    }
    r = g_nccl.GroupEnd();
    if (r) {
        *err = nccl_msg("ncclGroupEnd", r);
        return MOA_ERR_NCCL;
    }
    return MOA_OK;
}

// General point-to-point round (the N2 redistributions, redist.cu): this rank sends
// send_n[d] elements from send[d] to every rank d and receives recv_n[s] elements into
// recv[s] from every rank s, in one NCCL group; the self entry is a device copy.
// Counts of 0 skip the pair (scatter / gather rounds touch only rank 0's pairs).
int dist_sendrecv(const double2 *const *send, const int64_t *send_n, double2 *const *recv, const int64_t *recv_n,
                  int p, int rank, cudaStream_t s, std::string *err) {
    if (!g_comm) {
        *err = "no communicator (moa_dist_init)";
        return MOA_ERR_NO_DIST;
    }
    if (send_n[rank] != recv_n[rank]) {
        *err = "self send and receive counts differ";
        return MOA_ERR_INVALID_ARG;
    }
    if (send_n[rank] > 0) {
        cudaError_t ce = cudaMemcpyAsync(recv[rank], send[rank], send_n[rank] * sizeof(double2),
                                         cudaMemcpyDeviceToDevice, s);
        if (ce != cudaSuccess) {
            *err = std::string("self copy failed: ") + cudaGetErrorString(ce);
            return MOA_ERR_CUDA;
        }
    }
    ncclResult_t r = g_nccl.GroupStart();
    if (r) {
        *err = nccl_msg("ncclGroupStart", r);
        return MOA_ERR_NCCL;
    }
    for (int o = 1; o < p; ++o) {
        const int peer = (rank + o) % p, from = (rank - o + p) % p;
        if (send_n[peer] > 0) r = g_nccl.Send(send[peer], (size_t)send_n[peer] * 2, kNcclFloat64, peer, g_comm, s);
        if (!r && recv_n[from] > 0)
            r = g_nccl.Recv(recv[from], (size_t)recv_n[from] * 2, kNcclFloat64, from, g_comm, s);
        if (r) {
            g_nccl.GroupEnd();
            *err = nccl_msg("ncclSend/ncclRecv", r);
            return MOA_ERR_NCCL;
        }
    }
    r = g_nccl.GroupEnd();
    if (r) {
        *err = nccl_msg("ncclGroupEnd", r);
        return MOA_ERR_NCCL;
    }
    return MOA_OK;
}

// Stream-ordered barrier of all ranks (the P2P exchange's only collective): an
// 8-byte all-reduce completes on a rank only after every rank has enqueued it,
// i.e. after every rank's preceding kernels (the fused push) have finished.
int dist_barrier(cudaStream_t s, std::string *err) {
    if (!g_comm) {
        *err = "no communicator (moa_dist_init)";
        return MOA_ERR_NO_DIST;
    }
    if (!g_barrier_buf && cudaMalloc((void **)&g_barrier_buf, sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        *err = "barrier buffer allocation failed";
        return MOA_ERR_OOM;
    }
    ncclResult_t r = g_nccl.AllReduce(g_barrier_buf, g_barrier_buf, 1, kNcclFloat64, 0 /* sum */, g_comm, s);
    if (r) {
        *err = nccl_msg("ncclAllReduce (barrier)", r);
        return MOA_ERR_NCCL;
    }
    return MOA_OK;
}

// all-gather `bytes` per rank between device buffers, synchronous (plan setup only)
int dist_allgather_sync(const void *send_dev, void *recv_dev, size_t bytes, cudaStream_t s, std::string *err) {
    if (!g_comm) {
        *err = "no communicator (moa_dist_init)";
        return MOA_ERR_NO_DIST;
    }
    ncclResult_t r = g_nccl.AllGather(send_dev, recv_dev, bytes, 1 /* ncclUint8 */, g_comm, s);
    if (r) {
        *err = nccl_msg("ncclAllGather", r);
        return MOA_ERR_NCCL;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        *err = "stream synchronize after ncclAllGather failed";
        return MOA_ERR_CUDA;
    }
    return MOA_OK;
}

}  // namespace moa

extern "C" {

static int dist_fail(int code, const std::string &m) { return moa::fail(code, "%s", m.c_str()); }

int moa_dist_unique_id(void *id_out_128B) {
    std::string err;
    if (!id_out_128B) return dist_fail(MOA_ERR_INVALID_ARG, "NULL id buffer");
    int rc = load_nccl(&err);
    if (rc) return dist_fail(rc, err);
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r) return dist_fail(MOA_ERR_NCCL, nccl_msg("ncclGetUniqueId", r));
    memcpy(id_out_128B, &id, sizeof id);
    return MOA_OK;
}

int moa_dist_init(int rank, int p, const void *id_128B) {
    std::string err;
    if (!id_128B || p < 1 || rank < 0 || rank >= p)
        return dist_fail(MOA_ERR_INVALID_ARG, "bad rank/p/id for moa_dist_init");
    if (g_comm) return dist_fail(MOA_ERR_INVALID_ARG, "moa_dist_init called twice (finalize first)");
    int rc = load_nccl(&err);
    if (rc) return dist_fail(rc, err);
    ncclUniqueId id;
    memcpy(&id, id_128B, sizeof id);
    ncclComm_t c = nullptr;
    ncclResult_t r = g_nccl.CommInitRank(&c, p, id, rank);
    if (r) return dist_fail(MOA_ERR_NCCL, nccl_msg("ncclCommInitRank", r));
    g_comm = c;
    g_rank = rank;
    g_size = p;
    return MOA_OK;
}

int moa_dist_finalize(void) {
    if (g_barrier_buf) {
        cudaFree(g_barrier_buf);
        g_barrier_buf = nullptr;
    }
    if (g_comm) {
        g_nccl.CommDestroy(g_comm);
        g_comm = nullptr;
    }
    g_rank = -1;
    g_size = 0;
    return MOA_OK;
}

}  // extern "C"
