// comm.h -- internal: the communicator behind the C-ABI's peel_comm handle, shared by the
// partitioned k-core (dist.cu) and the cell-partitioned IBLT (iblt_dist.cu).  Three kinds:
//   NCCL     one process per GPU, collectives and grouped send/recv over NVLink;
//   host     one process per rank, collectives through caller-supplied host callbacks
//            (peel_comm_init_host; e.g. torch.distributed gloo) with device<->host staging:
//            the per-rank protocol of the NCCL path, runnable with several ranks on one GPU
//            because no kernel ever waits on another rank;
//   virtual  P shards inside one process on one GPU, exchanges as device copies.
// The rank code of dist.cu / iblt_dist.cu is the same for NCCL and host communicators: it
// calls the comm_* collectives below, which dispatch on the kind.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include "peel.h"

struct peel_comm {
    int P;          // number of shards (ranks)
    int rank;       // this process's rank, -1 for virtual shards
    bool virt;      // virtual shards of one GPU
    bool host;      // host-staged transport (callbacks)
    ncclComm_t nccl;
    peel_host_allreduce_fn h_allreduce;
    peel_host_allgather_fn h_allgather;
    peel_host_alltoallv_fn h_alltoallv;
    void *h_ctx;
    char *pin;          // pinned staging of the host transport (grown on demand)
    size_t pin_bytes;
};

namespace peel {
typedef unsigned long long ull;
void set_cuda_error(cudaError_t e, const char *where);
inline void nccl_error(ncclResult_t r) { set_cuda_error(cudaErrorUnknown, ncclGetErrorString(r)); }

// All collectives below are for rank communicators (NCCL or host), are called by every rank
// in the same order, and return when their results are usable on the host (host buffers) or
// on stream s (device buffers).  dstage: >= 8 P + 8 words of device scratch.
//   allreduce_sum   vals[count] (host) <- elementwise sum over ranks
//   allgather_u64   recv[P count] (host) <- every rank's send[count], in rank order
//   allgather_dev   recv_dev[P bytes] <- every rank's send_dev[bytes] (send_dev may be
//                   recv_dev + rank bytes: in place)
//   alltoallv       rank me sends send[d][0 .. sbytes[d]) to every d != me and receives
//                   rbytes[q] bytes from every q != me, packed in increasing q into recv
peel_status comm_allreduce_sum(peel_comm *c, ull *vals, int count, ull *dstage, cudaStream_t s);
peel_status comm_allgather_u64(peel_comm *c, const ull *send, ull *recv, int count, ull *dstage, cudaStream_t s);
peel_status comm_allgather_dev(peel_comm *c, const void *send_dev, void *recv_dev, size_t bytes, cudaStream_t s);
peel_status comm_alltoallv(peel_comm *c, const char *const *send, const ull *sbytes, char *recv, const ull *rbytes,
                           cudaStream_t s);
// Entry agreement of a partitioned call: every rank reports its local validation status;
// returns it if non-OK, PEEL_EPEER if another rank's was, else PEEL_OK -- so a rank that
// rejects its arguments never leaves the others blocked in the first collective.  Virtual
// communicators return `local` unchanged.
peel_status comm_agree(peel_comm *c, peel_status local, cudaStream_t s);
// stream sync after NCCL work with a watchdog (asynchronous NCCL errors, PEEL_NCCL_TIMEOUT_S):
// on either the communicator is aborted and PEEL_ENCCL returned; other kinds: a plain sync
peel_status comm_sync(peel_comm *c, cudaStream_t s);

// Test hook (PEEL_FAULT="rank:round"): true when this rank must fail in that round, to
// exercise the error protocol of the partitioned calls.
bool comm_fault(const peel_comm *c, uint32_t round);
}  // namespace peel

#define PEEL_NCCL(call)                       \
    do {                                      \
        ncclResult_t _r = (call);             \
        if (_r != ncclSuccess) {              \
            peel::nccl_error(_r);             \
            return PEEL_ENCCL;                \
        }                                     \
    } while (0)
