// comm.cu -- the communicator (comm.h): NCCL, host-staged (callbacks) and virtual shards, and
// the collectives the partitioned paths use ("one all-to-all ... one-word
// allreduce" per round).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include <chrono>
#include <thread>

#include "comm.h"
#include "common.cuh"

namespace peel {

static peel_status host_fail(const char *what) {
    char buf[128];
    snprintf(buf, sizeof buf, "host transport callback %s", what);
    set_cuda_error(cudaErrorUnknown, buf);
    return PEEL_ENCCL;
}

// pinned staging of at least `bytes`
static peel_status pin(peel_comm *c, size_t bytes) {
    if (c->pin_bytes >= bytes) return PEEL_OK;
    if (c->pin) cudaFreeHost(c->pin);
    c->pin = nullptr;
    c->pin_bytes = 0;
    size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 2;
    PEEL_CUDA(cudaMallocHost((void **)&c->pin, want));
    c->pin_bytes = want;
    return PEEL_OK;
}

// Stream sync after NCCL work, with a watchdog: polls the stream and ncclCommGetAsyncError,
// and aborts the communicator (every later call on it fails with PEEL_ENCCL) on an
// asynchronous NCCL error or after PEEL_NCCL_TIMEOUT_S seconds (default 600) -- a peer that
// died or left mid-protocol cannot hang this rank forever.  Other communicators: a plain sync.
static double nccl_timeout_s() {
    const char *e = getenv("PEEL_NCCL_TIMEOUT_S");
    const double t = e ? atof(e) : 600.0;
    return t > 0 ? t : 600.0;
}

peel_status comm_sync(peel_comm *c, cudaStream_t s) {
    if (c->virt || c->host) {
        PEEL_CUDA(cudaStreamSynchronize(s));
        return PEEL_OK;
    }
    if (!c->nccl) {
        set_cuda_error(cudaErrorUnknown, "NCCL communicator aborted");
        return PEEL_ENCCL;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = nccl_timeout_s();
    for (uint32_t it = 0;; it++) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return PEEL_OK;
        if (q != cudaErrorNotReady) {
            set_cuda_error(q, "stream sync");
            return PEEL_ECUDA;
        }
        ncclResult_t ar = ncclSuccess;
        const ncclResult_t gr = ncclCommGetAsyncError(c->nccl, &ar);
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (gr != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress) || el > limit) {
            set_cuda_error(cudaErrorUnknown, el > limit ? "NCCL watchdog: timeout, communicator aborted"
                                                        : "NCCL asynchronous error, communicator aborted");
            ncclCommAbort(c->nccl);
            c->nccl = nullptr;
            return PEEL_ENCCL;
        }
        if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

peel_status comm_allreduce_sum(peel_comm *c, ull *vals, int count, ull *dstage, cudaStream_t s) {
    if (c->host) {
        if (c->h_allreduce(c->h_ctx, (uint64_t *)vals, (uint64_t)count)) return host_fail("allreduce");
        return PEEL_OK;
    }
    PEEL_CUDA(cudaMemcpyAsync(dstage, vals, sizeof(ull) * count, cudaMemcpyHostToDevice, s));
    if (!c->nccl) return comm_sync(c, s);
    PEEL_NCCL(ncclAllReduce(dstage, dstage, count, ncclUint64, ncclSum, c->nccl, s));
    // wait with the watchdog BEFORE the copy back: a copy to pageable memory blocks inside
    // the runtime until the stream drains, where no watchdog could see a dead peer
    const peel_status ws = comm_sync(c, s);
    if (ws != PEEL_OK) return ws;
    PEEL_CUDA(cudaMemcpy(vals, dstage, sizeof(ull) * count, cudaMemcpyDeviceToHost));
    return PEEL_OK;
}

peel_status comm_allgather_u64(peel_comm *c, const ull *send, ull *recv, int count, ull *dstage, cudaStream_t s) {
    if (c->host) {
        if (c->h_allgather(c->h_ctx, send, recv, sizeof(ull) * count)) return host_fail("allgather");
        return PEEL_OK;
    }
    ull *mine = dstage + (size_t)c->rank * count;
    PEEL_CUDA(cudaMemcpyAsync(mine, send, sizeof(ull) * count, cudaMemcpyHostToDevice, s));
    if (!c->nccl) return comm_sync(c, s);
    PEEL_NCCL(ncclAllGather(mine, dstage, count, ncclUint64, c->nccl, s));
    const peel_status ws = comm_sync(c, s);  // before the (blocking) copy back, as above
    if (ws != PEEL_OK) return ws;
    PEEL_CUDA(cudaMemcpy(recv, dstage, sizeof(ull) * count * c->P, cudaMemcpyDeviceToHost));
    return PEEL_OK;
}

peel_status comm_allgather_dev(peel_comm *c, const void *send_dev, void *recv_dev, size_t bytes, cudaStream_t s) {
    if (c->host) {
        peel_status st = pin(c, bytes * (c->P + 1));
        if (st != PEEL_OK) return st;
        char *mine = c->pin + bytes * c->P;
        PEEL_CUDA(cudaMemcpyAsync(mine, send_dev, bytes, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaStreamSynchronize(s));
        if (c->h_allgather(c->h_ctx, mine, c->pin, bytes)) return host_fail("allgather");
        PEEL_CUDA(cudaMemcpyAsync(recv_dev, c->pin, bytes * c->P, cudaMemcpyHostToDevice, s));
        return PEEL_OK;
    }
    if (!c->nccl) return comm_sync(c, s);
    PEEL_NCCL(ncclAllGather(send_dev, recv_dev, bytes, ncclUint8, c->nccl, s));
    return PEEL_OK;
}

peel_status comm_alltoallv(peel_comm *c, const char *const *send, const ull *sbytes, char *recv, const ull *rbytes,
                           cudaStream_t s) {
    const int P = c->P, me = c->rank;
    if (c->host) {
        ull stot = 0, rtot = 0;
        for (int q = 0; q < P; q++)
            if (q != me) { stot += sbytes[q]; rtot += rbytes[q]; }
        peel_status st = pin(c, stot + rtot);
        if (st != PEEL_OK) return st;
        char *sp = c->pin, *rp = c->pin + stot;
        std::vector<uint64_t> sb(P, 0), rb(P, 0);
        ull o = 0;
        for (int q = 0; q < P; q++) {
            if (q == me || !sbytes[q]) continue;
            PEEL_CUDA(cudaMemcpyAsync(sp + o, send[q], sbytes[q], cudaMemcpyDeviceToHost, s));
            sb[q] = sbytes[q];
            o += sbytes[q];
        }
        for (int q = 0; q < P; q++) rb[q] = q == me ? 0 : rbytes[q];
        PEEL_CUDA(cudaStreamSynchronize(s));
        if (c->h_alltoallv(c->h_ctx, sp, sb.data(), rp, rb.data())) return host_fail("alltoallv");
        if (rtot) PEEL_CUDA(cudaMemcpyAsync(recv, rp, rtot, cudaMemcpyHostToDevice, s));
        // the staging is reused by the next collective: wait for the copy out of it
        PEEL_CUDA(cudaStreamSynchronize(s));
        return PEEL_OK;
    }
    if (!c->nccl) return comm_sync(c, s);
    PEEL_NCCL(ncclGroupStart());
    ull off = 0;
    for (int q = 0; q < P; q++) {
        if (q == me) continue;
        if (rbytes[q]) {
            ncclResult_t r = ncclRecv(recv + off, rbytes[q], ncclUint8, q, c->nccl, s);
            if (r != ncclSuccess) { ncclGroupEnd(); nccl_error(r); return PEEL_ENCCL; }
        }
        off += rbytes[q];
    }
    for (int q = 0; q < P; q++) {
        if (q == me || !sbytes[q]) continue;
        ncclResult_t r = ncclSend(send[q], sbytes[q], ncclUint8, q, c->nccl, s);
        if (r != ncclSuccess) { ncclGroupEnd(); nccl_error(r); return PEEL_ENCCL; }
    }
    PEEL_NCCL(ncclGroupEnd());
    return PEEL_OK;
}

peel_status comm_agree(peel_comm *c, peel_status local, cudaStream_t s) {
    if (c->virt) return local;
    // NCCL: a local validation failure may be a bad stream or workspace; the agreement word
    // goes through a small cudaMalloc'd scratch so it never touches the caller's buffers
    ull w[1] = {local != PEEL_OK ? 1ull : 0ull};
    peel_status st;
    if (c->host) {
        st = comm_allreduce_sum(c, w, 1, nullptr, s);
    } else {
        static ull *scratch[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64) return PEEL_EINVAL;
        if (!scratch[dev]) PEEL_CUDA(cudaMalloc((void **)&scratch[dev], 64));
        st = comm_allreduce_sum(c, w, 1, scratch[dev], s);
    }
    if (local != PEEL_OK) return local;
    if (st != PEEL_OK) return st;
    return w[0] ? PEEL_EPEER : PEEL_OK;
}

bool comm_fault(const peel_comm *c, uint32_t round) {
    const char *e = getenv("PEEL_FAULT");
    if (!e || c->virt) return false;
    int fr = -1;
    unsigned ft = 0;
    if (sscanf(e, "%d:%u", &fr, &ft) != 2) return false;
    return fr == c->rank && ft == round;
}

}  // namespace peel

using namespace peel;

static peel_comm *new_comm(int P, int rank) {
    peel_comm *c = new peel_comm;
    memset(c, 0, sizeof *c);
    c->P = P;
    c->rank = rank;
    return c;
}

extern "C" peel_status peel_comm_unique_id(void *id128) {
    if (!id128) return PEEL_EINVAL;
    ncclUniqueId id;
    PEEL_NCCL(ncclGetUniqueId(&id));
    memcpy(id128, &id, sizeof(id));
    return PEEL_OK;
}

extern "C" peel_status peel_comm_init(const void *id128, int nranks, int rank, peel_comm **out) {
    if (!id128 || !out || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) return PEEL_EINVAL;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    peel_comm *c = new_comm(nranks, rank);
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        peel::nccl_error(r);
        return PEEL_ENCCL;
    }
    *out = c;
    return PEEL_OK;
}

extern "C" peel_status peel_comm_init_host(int nranks, int rank, peel_host_allreduce_fn allreduce,
                                           peel_host_allgather_fn allgather, peel_host_alltoallv_fn alltoallv,
                                           void *ctx, peel_comm **out) {
    if (!out || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks || !allreduce || !allgather || !alltoallv)
        return PEEL_EINVAL;
    peel_comm *c = new_comm(nranks, rank);
    c->host = true;
    c->h_allreduce = allreduce;
    c->h_allgather = allgather;
    c->h_alltoallv = alltoallv;
    c->h_ctx = ctx;
    *out = c;
    return PEEL_OK;
}

extern "C" peel_status peel_comm_init_virtual(int nshards, peel_comm **out) {
    if (!out || nshards < 1 || nshards > 8) return PEEL_EINVAL;
    peel_comm *c = new_comm(nshards, -1);
    c->virt = true;
    *out = c;
    return PEEL_OK;
}

extern "C" void peel_comm_destroy(peel_comm *c) {
    if (!c) return;
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->pin) cudaFreeHost(c->pin);
    delete c;
}
