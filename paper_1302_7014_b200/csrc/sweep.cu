// sweep.cu -- independent-trial sweeps (the paper's simulation protocol,
// "we ran the program 1000 times ... and computed the average number of rounds").
//
// A batch of B trials is peeled as ONE disjoint-union hypergraph: trial b's vertices are
// [b n, (b+1) n) and its edges are G^r_{n,m_b}(seed_b) shifted by b n.  Round-synchronous
// peeling of a disjoint union is exactly the B independent synchronous peels run in
// lockstep (F_t of the union = the union of the trials' F_t), so one peel_kcore call over
// the union -- with its binned build, persistent round loop and all -- computes every
// trial.  Per trial: rounds = max over its vertices of the removal round, core = number
// of its vertices never removed (a segmented reduction over peel_round / core_mask).
#include <stdlib.h>

#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace peel {

static inline size_t al2(size_t x) { return (x + 255) & ~(size_t)255; }

// per trial b = blockIdx.y: max removal round and core size over its n vertices; blocks
// blockIdx.x split the trial into SR_CH-vertex chunks and combine with atomics (outputs zeroed)
static constexpr uint32_t SR_CH = 8192;

__global__ void __launch_bounds__(256) sweep_reduce_kernel(const uint32_t *__restrict__ peel_round,
                                                           const uint8_t *__restrict__ mask, uint64_t n,
                                                           ull *out_rounds, ull *out_core) {
    const uint64_t b = blockIdx.y;
    const uint64_t lo = (uint64_t)blockIdx.x * SR_CH, hi = min(n, lo + SR_CH);
    const uint32_t *pr = peel_round + b * n;
    const uint8_t *mk = mask + b * n;
    uint32_t mx = 0;
    ull core = 0;
    for (uint64_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
        mx = max(mx, __ldcs(pr + v));
        core += __ldcs(mk + v);
    }
    __shared__ uint32_t smx[8];
    __shared__ ull score[8];
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        core += __shfl_xor_sync(0xffffffffu, core, o);
    }
    if ((threadIdx.x & 31) == 0) { smx[threadIdx.x >> 5] = mx; score[threadIdx.x >> 5] = core; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; w++) { mx = max(mx, smx[w]); core += score[w]; }
        if (mx) atomicMax(out_rounds + b, (ull)mx);
        if (core) atomicAdd(out_core + b, core);
    }
}

struct SweepLayout {
    size_t edges, mask, pr, res, par, kws, total;
    size_t kws_bytes;
};

static SweepLayout sweep_layout(uint64_t n, uint64_t max_m, uint32_t r, uint32_t k, uint32_t batch) {
    SweepLayout L;
    size_t o = 0;
    L.edges = o; o += al2(sizeof(uint32_t) * r * max_m * batch);
    L.mask = o; o += al2(n * batch);
    L.pr = o; o += al2(sizeof(uint32_t) * n * batch);
    L.res = o; o += al2(sizeof(ull) * 2 * batch);
    L.par = o; o += al2(sizeof(ull) * (2 * batch + 1));  // trial m prefix sums and seeds (device copy)
    L.kws_bytes = peel_kcore_workspace_bytes(n * batch, max_m * batch, r, k, 0);
    L.kws = o; o += al2(L.kws_bytes);
    L.total = L.kws_bytes ? o : 0;
    return L;
}

}  // namespace peel

using namespace peel;

// Batches run on NW host worker threads, each with its own stream and workspace slice: the
// GPU overlaps one batch's latency-bound tail rounds with another batch's build
// (PEEL_SWEEP_WORKERS, default 2)
static uint32_t sweep_workers() {
    const char *e = getenv("PEEL_SWEEP_WORKERS");
    const int w = e ? atoi(e) : 2;
    return (uint32_t)(w < 1 ? 1 : (w > 8 ? 8 : w));
}

extern "C" size_t peel_sweep_workspace_bytes(uint64_t n, uint64_t max_m, uint32_t r, uint32_t k, uint32_t batch) {
    if (batch == 0 || batch > 1024 || n < r || n * batch > (1ull << 32) || max_m * batch >= (1ull << 32)) return 0;
    return sweep_layout(n, max_m, r, k, batch).total * sweep_workers();
}

extern "C" peel_status peel_sweep(uint64_t n, uint32_t r, uint32_t k, const uint64_t *m, const uint64_t *seeds,
                                  uint64_t ntrials, uint32_t batch, uint32_t *out_rounds, uint64_t *out_core,
                                  void *workspace, size_t ws_bytes, void *stream) {
    if (!m || !seeds || !out_rounds || !out_core || !workspace || batch == 0 || batch > 1024 || r < 2 || r > 8 || n < r)
        return PEEL_EINVAL;
    uint64_t max_m = 0;
    for (uint64_t t = 0; t < ntrials; t++) max_m = m[t] > max_m ? m[t] : max_m;
    if (n * batch > (1ull << 32) || max_m * batch >= (1ull << 32)) return PEEL_EINVAL;
    SweepLayout L = sweep_layout(n, max_m, r, k, batch);
    if (!L.total) return PEEL_EINVAL;
    const uint64_t nbatches = (ntrials + batch - 1) / batch;
    uint32_t NW = sweep_workers();
    if (ws_bytes < L.total * NW) {
        if (ws_bytes < L.total) return PEEL_ENOMEM;
        NW = 1;  // a workspace sized for one worker (the caller's own query of another setting)
    }
    if (NW > nbatches) NW = (uint32_t)(nbatches ? nbatches : 1);
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    PEEL_CUDA(cudaGetDevice(&dev));
    prof_begin_call();
    prof_hold(true);  // the batches' peel_kcore calls report as this one call
    struct Release {
        ~Release() {
            prof_hold(false);
            prof_collect();
        }
    } release;
    // worker w: batches w, w + NW, ...; its own stream (after the caller's stream's prior work)
    cudaEvent_t start = nullptr;
    PEEL_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    PEEL_CUDA(cudaEventRecord(start, s));
    std::vector<peel_status> st(NW, PEEL_OK);
    std::vector<std::string> err(NW);
    auto worker = [&](uint32_t w) {
        if (cudaSetDevice(dev) != cudaSuccess) { st[w] = PEEL_ECUDA; return; }
        cudaStream_t ws_s = nullptr;
        if (cudaStreamCreateWithFlags(&ws_s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamWaitEvent(ws_s, start, 0) != cudaSuccess) {
            st[w] = PEEL_ECUDA;
            return;
        }
        char *ws = (char *)workspace + (size_t)w * L.total;
        uint32_t *edges = (uint32_t *)(ws + L.edges);
        uint8_t *mask = (uint8_t *)(ws + L.mask);
        uint32_t *pr = (uint32_t *)(ws + L.pr);
        ull *res = (ull *)(ws + L.res);
        ull *par = (ull *)(ws + L.par);
        std::vector<ull> hres(2 * batch), hpar(2 * batch + 1);
        auto run = [&]() -> peel_status {
            for (uint64_t bi = w; bi < nbatches; bi += NW) {
                const uint64_t t0 = bi * batch;
                const uint32_t B = (uint32_t)(ntrials - t0 < batch ? ntrials - t0 : batch);
                // one generator launch for the batch: prefix sums of m and the seeds go to the device
                hpar[0] = 0;
                for (uint32_t b = 0; b < B; b++) {
                    hpar[b + 1] = hpar[b] + m[t0 + b];
                    hpar[batch + 1 + b] = seeds[t0 + b];
                }
                const uint64_t off = hpar[B];
                PEEL_CUDA(cudaMemcpyAsync(par, hpar.data(), sizeof(ull) * (2 * batch + 1), cudaMemcpyHostToDevice, ws_s));
                peel_status st2 = launch_gen_batch(n, r, B, (const uint64_t *)par, (const uint64_t *)par + batch + 1,
                                                   off, edges, ws_s);
                if (st2 != PEEL_OK) return st2;
                uint32_t rounds = 0;
                st2 = peel_kcore(edges, n * B, off, r, k, 0, mask, &rounds, nullptr, nullptr, 0, pr, ws + L.kws,
                                 L.kws_bytes, ws_s);
                if (st2 != PEEL_OK && st2 != PEEL_ETRUNC) return st2;
                PEEL_CUDA(cudaMemsetAsync(res, 0, sizeof(ull) * 2 * batch, ws_s));
                {
                    ProfScope ps("sweep_reduce", ws_s);
                    sweep_reduce_kernel<<<dim3((unsigned)((n + SR_CH - 1) / SR_CH), B), 256, 0, ws_s>>>(pr, mask, n, res,
                                                                                                    res + batch);
                }
                PEEL_CUDA(cudaGetLastError());
                PEEL_CUDA(cudaMemcpyAsync(hres.data(), res, sizeof(ull) * 2 * batch, cudaMemcpyDeviceToHost, ws_s));
                PEEL_CUDA(cudaStreamSynchronize(ws_s));
                for (uint32_t b = 0; b < B; b++) {
                    out_rounds[t0 + b] = (uint32_t)hres[b];
                    out_core[t0 + b] = hres[batch + b];
                }
            }
            return PEEL_OK;
        };
        st[w] = run();
        if (st[w] != PEEL_OK) err[w] = peel_last_cuda_error();
        cudaStreamSynchronize(ws_s);
        cudaStreamDestroy(ws_s);
    };
    std::vector<std::thread> th;
    for (uint32_t w = 1; w < NW; w++) th.emplace_back(worker, w);
    worker(0);
    for (auto &x : th) x.join();
    cudaEventDestroy(start);
    for (uint32_t w = 0; w < NW; w++)
        if (st[w] != PEEL_OK) return st[w];
    return PEEL_OK;
}
