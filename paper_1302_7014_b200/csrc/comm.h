// comm.h -- internal: the communicator behind the C-ABI's peel_comm handle (NCCL ranks or
// virtual shards of one GPU), shared by the partitioned k-core (dist.cu) and the
// cell-partitioned IBLT (iblt_dist.cu).
#pragma once
#include <nccl.h>

#include "peel.h"

struct peel_comm {
    int P;          // number of shards (ranks)
    int rank;       // this process's rank (NCCL), -1 for virtual shards
    bool virt;
    ncclComm_t nccl;
};

namespace peel {
void set_cuda_error(cudaError_t e, const char *where);
inline void nccl_error(ncclResult_t r) { set_cuda_error(cudaErrorUnknown, ncclGetErrorString(r)); }
}  // namespace peel

#define PEEL_NCCL(call)                       \
    do {                                      \
        ncclResult_t _r = (call);             \
        if (_r != ncclSuccess) {              \
            peel::nccl_error(_r);             \
            return PEEL_ENCCL;                \
        }                                     \
    } while (0)
