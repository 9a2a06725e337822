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
#include "genrow.cuh"

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

// ---- per-trial groups (k = 2, r <= 4, n <= 2^22: the paper's protocol, C5s) ------------------
// A trial of the protocol (n = 10^6) has a 4 MB working set once its state is one 32-bit word
// per vertex, so the whole peel stays in L2 if only ~16 trials are in flight.  NG groups of G
// co-resident CTAs (one cooperative launch) take trials off a counter; a group peels its trial
// with group barriers (one L2 counter) between phases and rounds, and regenerates a killed
// edge's row from (seed, e) -- G^r_{n,m} is a pure function of it (genrow.cuh), so no edge list
// is stored.  The schedule is kcore.cu's (the crossing rule of DESIGN §5):
//   state[v] = (Σ incident alive edge ids mod 2^(32-CB)) << CB | count        (count < 2^CB)
// m <= 2^(32-CB), so a count-1 vertex's id field IS its edge.  A count reaching 2^CB would carry
// into the id field: the scan checks Σ count == r m and flags the trial, and the host peels a
// flagged trial on the union path.  Per trial: rounds = rounds with F_t non-empty, core =
// vertices with count >= k after the build minus the crossings of every round.
static constexpr int SG_BLOCK = 512;
#ifndef PEEL_SG_MINB
#define PEEL_SG_MINB 3
#endif
static constexpr int SG_QCAP = 2048;
static constexpr uint32_t SG_CHUNK = 65536;  // trials per launch (device result arrays)

struct __align__(128) SGroupCtl {
    unsigned bar;    // barrier arrivals (monotonic over the launch)
    unsigned trial;  // the group's trial
    ull cnt[3];      // frontier entries of round t at cnt[t % 3]
    ull sum, live, nf1;
};

struct SGArgs {
    uint64_t n;
    uint32_t k, cb, G, ntrials;
    const uint64_t *m, *seeds;
    uint32_t *out_rounds, *flag;
    ull *out_core;
    uint32_t *state;  // per group: sstride words
    uint32_t *alive;  // per group: astride words
    uint32_t *list;   // per group: 2 lists of n entries (lstride words)
    uint64_t sstride, astride, lstride;
    SGroupCtl *ctl;
    unsigned *next;
};

// barrier of the group's G CTAs (co-resident: cooperative launch); every thread calls it
__device__ __forceinline__ void group_sync(unsigned *bar, unsigned &target, unsigned G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        target += G;
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) {}
    }
    __syncthreads();
}

template <int R>
__global__ void __launch_bounds__(SG_BLOCK, PEEL_SG_MINB) sweep_group_kernel(SGArgs a) {
    typedef BlockQueueT<uint32_t, SG_QCAP, SG_BLOCK> Q;
    __shared__ Q bq;
    __shared__ unsigned s_trial;
    const uint32_t g = blockIdx.x / a.G, q = blockIdx.x % a.G;
    SGroupCtl *c = a.ctl + g;
    uint32_t *st = a.state + g * a.sstride;
    uint32_t *alive = a.alive + g * a.astride;
    uint32_t *L0 = a.list + g * a.lstride, *L1 = L0 + a.n;
    const uint64_t tg = (uint64_t)q * SG_BLOCK + threadIdx.x, nthr = (uint64_t)a.G * SG_BLOCK;
    const uint64_t n = a.n;
    const uint32_t CB = a.cb, cmask = (1u << CB) - 1u, k = a.k;
    unsigned target = 0;
    bq_init(bq);
    int slot = 0;
    for (;;) {
        if (q == 0 && threadIdx.x == 0) {
            c->trial = atomicAdd(a.next, 1u);
            c->cnt[0] = c->cnt[1] = c->cnt[2] = 0ull;
            c->sum = c->live = c->nf1 = 0ull;
        }
        group_sync(&c->bar, target, a.G);
        if (threadIdx.x == 0) s_trial = *(volatile unsigned *)&c->trial;
        __syncthreads();
        const uint32_t T = s_trial;
        if (T >= a.ntrials) break;  // uniform over the group
        const uint64_t m = a.m[T], seed = a.seeds[T];
        const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
        // zero the state; alive bits of edges [0, m)
        {
            uint4 *z = reinterpret_cast<uint4 *>(st);
            for (uint64_t i = tg; i < (n + 3) / 4; i += nthr) z[i] = make_uint4(0u, 0u, 0u, 0u);
            const uint64_t aw = (m + 31) / 32;
            for (uint64_t i = tg; i < aw; i += nthr)
                alive[i] = (i == aw - 1 && (m & 31)) ? ((1u << (m & 31)) - 1u) : ~0u;
        }
        group_sync(&c->bar, target, a.G);
        // build: r increments per edge (fire-and-forget REDs into the L2-resident state)
        for (uint64_t e = tg; e < m; e += nthr) {
            uint32_t u[R];
            gen_one_edge<R>(e, n, k0, k1, u);
            const uint32_t inc = ((uint32_t)e << CB) + 1u;
            #pragma unroll
            for (int j = 0; j < R; j++) asm volatile("red.global.add.u32 [%0], %1;" ::"l"(st + u[j]), "r"(inc) : "memory");
        }
        group_sync(&c->bar, target, a.G);
        // scan: F_1 (count < k), its entries (count 1), the live set, the overflow check
        {
            ull sum = 0, live = 0, nf = 0;
            for (uint64_t v0 = (uint64_t)q * SG_BLOCK; v0 < n; v0 += nthr) {
                const uint64_t v = v0 + threadIdx.x;
                if (v < n) {
                    const uint32_t cnt = __ldcg(st + v) & cmask;
                    sum += cnt;
                    if (cnt >= k) live++;
                    else {
                        nf++;
                        if (cnt == 1u) bq_push(bq, slot, (uint32_t)v, L0, &c->cnt[1]);
                    }
                }
                bq_flush(bq, slot, L0, &c->cnt[1]);
                slot ^= 1;
            }
            block_add<SG_BLOCK>(&c->sum, sum);
            block_add<SG_BLOCK>(&c->live, live);
            block_add<SG_BLOCK>(&c->nf1, nf);
        }
        group_sync(&c->bar, target, a.G);
        const ull S = ld_cg_u64(&c->sum), LIVE = ld_cg_u64(&c->live), NF1 = ld_cg_u64(&c->nf1);
        const bool over = S != (ull)R * m;
        uint32_t rounds = NF1 ? 1u : 0u;
        ull crossed = 0;
        for (uint32_t t = 1; !over; t++) {
            const ull E = ld_cg_u64(&c->cnt[t % 3]);  // entries of F_t (t >= 2: |F_t|)
            if (E == 0) break;                          // uniform: read after the same barrier
            if (t >= 2) { rounds = t; crossed += E; }
            if (q == 0 && threadIdx.x == 0) c->cnt[(t + 2) % 3] = 0ull;  // read before the last barrier
            const uint32_t *Lc = (t & 1) ? L0 : L1;
            uint32_t *Ln = (t & 1) ? L1 : L0;
            ull *cn = &c->cnt[(t + 1) % 3];
            for (uint64_t i0 = (uint64_t)q * SG_BLOCK; i0 < E; i0 += nthr) {
                const uint64_t i = i0 + threadIdx.x;
                if (i < E) {
                    const uint32_t v = __ldcg(Lc + i);
                    // v has count 1 (its edge e alive at the round start) or 0 (e killed this
                    // round by another vertex of e): either way the test-and-clear decides
                    const uint32_t s = __ldcg(st + v);
                    const uint32_t e = s >> CB;
                    const uint32_t bit = 1u << (e & 31);
                    if ((s & cmask) && (atomicAnd(alive + (e >> 5), ~bit) & bit)) {
                        uint32_t u[R];
                        gen_one_edge<R>(e, n, k0, k1, u);
                        const uint32_t dec = 0u - ((e << CB) + 1u);
                        uint32_t old[R];
                        #pragma unroll
                        for (int j = 0; j < R; j++) old[j] = u[j] != v ? atomicAdd(st + u[j], dec) : 0u;
                        #pragma unroll
                        for (int j = 0; j < R; j++)
                            if (u[j] != v && (old[j] & cmask) == k) bq_push(bq, slot, u[j], Ln, cn);
                    }
                }
                bq_flush(bq, slot, Ln, cn);
                slot ^= 1;
            }
            group_sync(&c->bar, target, a.G);
        }
        group_sync(&c->bar, target, a.G);  // every CTA read the control block: it may be reset
        if (q == 0 && threadIdx.x == 0) {
            a.out_rounds[T] = rounds;
            a.out_core[T] = LIVE - crossed;
            a.flag[T] = over ? 1u : 0u;
        }
    }
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

// ---- the per-trial group path (host side)
// PEEL_SWEEP_GROUPS: 0 = off (every trial on the union path), N > 0 = N groups; unset = as many
// groups as fit PEEL_SWEEP_L2MB (default 100) MB of per-trial working set in L2.
static const uint32_t SG_NG_MAX = 512;

struct SGLayout {
    size_t ctl, next, par, res, state, alive, list, total;
    uint64_t sstride, astride, lstride;
    uint32_t NG, cb;
};

static uint32_t sg_bits(uint64_t x) {  // bits to hold values < x (x >= 1)
    uint32_t b = 1;
    while (b < 64 && (1ull << b) < x) b++;
    return b;
}

static bool sg_applicable(uint64_t n, uint64_t max_m, uint32_t r, uint32_t k) {
    const char *e = getenv("PEEL_SWEEP_GROUPS");
    if (e && atoi(e) == 0) return false;
    if (k != 2 || r < 2 || r > 4 || n < r || n > (1ull << 22)) return false;
    const uint32_t eb = sg_bits(max_m ? max_m : 1);
    return eb <= 28;  // at least 4 count bits
}

static SGLayout sg_layout(uint64_t n, uint64_t max_m) {
    SGLayout L;
    const char *e = getenv("PEEL_SWEEP_GROUPS");
    uint32_t ng;
    if (e && atoi(e) > 0) {
        ng = (uint32_t)atoi(e);
    } else {
        const char *l2 = getenv("PEEL_SWEEP_L2MB");
        // C5s (n = 10^6): 12 / 16 / 20 / 24 / 32 groups -> 514 / 482 / 471 / 488 / 542 ms
        const double budget = (l2 ? atof(l2) : 100.0) * 1048576.0;
        const double per = 4.0 * n * 1.25 + max_m / 8.0 + 4096.0;  // state, touched list part, alive bits
        ng = (uint32_t)(budget / per);
    }
    L.NG = ng < 1 ? 1 : (ng > SG_NG_MAX ? SG_NG_MAX : ng);
    L.cb = 32 - sg_bits(max_m ? max_m : 1);
    const char *cbe = getenv("PEEL_SWEEP_CB");  // tests: force a narrow count field (overflow path)
    if (cbe && atoi(cbe) > 0 && (uint32_t)atoi(cbe) < L.cb) L.cb = (uint32_t)atoi(cbe);
    L.sstride = (n + 63) & ~63ull;
    L.astride = (((max_m + 31) / 32) + 63) & ~63ull;
    L.lstride = (2 * n + 63) & ~63ull;
    size_t o = 0;
    L.ctl = o; o += al2(sizeof(SGroupCtl) * L.NG);
    L.next = o; o += al2(sizeof(unsigned));
    L.par = o; o += al2(sizeof(uint64_t) * 2 * SG_CHUNK);
    L.res = o; o += al2((sizeof(uint32_t) * 2 + sizeof(ull)) * SG_CHUNK);
    L.state = o; o += al2(sizeof(uint32_t) * L.sstride * L.NG);
    L.alive = o; o += al2(sizeof(uint32_t) * L.astride * L.NG);
    L.list = o; o += al2(sizeof(uint32_t) * L.lstride * L.NG);
    L.total = o;
    return L;
}

template <int R>
static peel_status sg_launch(SGArgs &a, uint32_t NG, cudaStream_t s) {
    int bps = 0;
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, sweep_group_kernel<R>, SG_BLOCK, 0));
    if (bps < 1) return PEEL_ECUDA;
    const uint32_t total = (uint32_t)(bps * num_sms());
    if (NG > total) NG = total;
    if (NG > a.ntrials) NG = a.ntrials;
    a.G = total / NG;
    void *args[] = {&a};
    ProfScope ps("sweep_groups", s);
    PEEL_CUDA(cudaLaunchCooperativeKernel((void *)sweep_group_kernel<R>, NG * a.G, SG_BLOCK, args, 0, s));
    return PEEL_OK;
}

// every trial on the group path; trials whose count field overflowed come back in `redo`
static peel_status sweep_groups(uint64_t n, uint32_t r, uint32_t k, const uint64_t *m, const uint64_t *seeds,
                                uint64_t ntrials, uint32_t *out_rounds, uint64_t *out_core, void *workspace,
                                const SGLayout &L, cudaStream_t s, std::vector<uint64_t> &redo) {
    char *ws = (char *)workspace;
    uint64_t *par = (uint64_t *)(ws + L.par);
    uint32_t *rr = (uint32_t *)(ws + L.res), *fl = rr + SG_CHUNK;
    ull *cr = (ull *)(fl + SG_CHUNK);
    std::vector<uint32_t> hr(SG_CHUNK), hf(SG_CHUNK);
    std::vector<ull> hc(SG_CHUNK);
    for (uint64_t t0 = 0; t0 < ntrials; t0 += SG_CHUNK) {
        const uint32_t B = (uint32_t)(ntrials - t0 < SG_CHUNK ? ntrials - t0 : SG_CHUNK);
        PEEL_CUDA(cudaMemcpyAsync(par, m + t0, sizeof(uint64_t) * B, cudaMemcpyHostToDevice, s));
        PEEL_CUDA(cudaMemcpyAsync(par + SG_CHUNK, seeds + t0, sizeof(uint64_t) * B, cudaMemcpyHostToDevice, s));
        PEEL_CUDA(cudaMemsetAsync(ws + L.ctl, 0, L.next + sizeof(unsigned) - L.ctl, s));
        SGArgs a;
        a.n = n; a.k = k; a.cb = L.cb; a.G = 1; a.ntrials = B;
        a.m = par; a.seeds = par + SG_CHUNK;
        a.out_rounds = rr; a.flag = fl; a.out_core = cr;
        a.state = (uint32_t *)(ws + L.state); a.alive = (uint32_t *)(ws + L.alive); a.list = (uint32_t *)(ws + L.list);
        a.sstride = L.sstride; a.astride = L.astride; a.lstride = L.lstride;
        a.ctl = (SGroupCtl *)(ws + L.ctl); a.next = (unsigned *)(ws + L.next);
        peel_status st = PEEL_EINVAL;
        switch (r) {
            case 2: st = sg_launch<2>(a, L.NG, s); break;
            case 3: st = sg_launch<3>(a, L.NG, s); break;
            case 4: st = sg_launch<4>(a, L.NG, s); break;
        }
        if (st != PEEL_OK) return st;
        PEEL_CUDA(cudaMemcpyAsync(hr.data(), rr, sizeof(uint32_t) * B, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaMemcpyAsync(hf.data(), fl, sizeof(uint32_t) * B, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaMemcpyAsync(hc.data(), cr, sizeof(ull) * B, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaStreamSynchronize(s));
        for (uint32_t b = 0; b < B; b++) {
            if (hf[b]) { redo.push_back(t0 + b); continue; }
            out_rounds[t0 + b] = hr[b];
            out_core[t0 + b] = hc[b];
        }
    }
    return PEEL_OK;
}

static size_t sweep_union_bytes(uint64_t n, uint64_t max_m, uint32_t r, uint32_t k, uint32_t batch) {
    if (batch == 0 || batch > 1024 || n < r || n * batch > (1ull << 32) || max_m * batch >= (1ull << 32)) return 0;
    return sweep_layout(n, max_m, r, k, batch).total * sweep_workers();
}

extern "C" size_t peel_sweep_workspace_bytes(uint64_t n, uint64_t max_m, uint32_t r, uint32_t k, uint32_t batch) {
    const size_t u = sweep_union_bytes(n, max_m, r, k, batch);
    if (!u || !sg_applicable(n, max_m, r, k)) return u;
    const size_t g = sg_layout(n, max_m).total;
    return g > u ? g : u;
}

static peel_status sweep_union(uint64_t n, uint32_t r, uint32_t k, const uint64_t *m, const uint64_t *seeds,
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

extern "C" peel_status peel_sweep(uint64_t n, uint32_t r, uint32_t k, const uint64_t *m, const uint64_t *seeds,
                                  uint64_t ntrials, uint32_t batch, uint32_t *out_rounds, uint64_t *out_core,
                                  void *workspace, size_t ws_bytes, void *stream) {
    if (!m || !seeds || !out_rounds || !out_core || !workspace || batch == 0 || batch > 1024 || r < 2 || r > 8 || n < r)
        return PEEL_EINVAL;
    uint64_t max_m = 0;
    for (uint64_t t = 0; t < ntrials; t++) max_m = m[t] > max_m ? m[t] : max_m;
    if (n * batch > (1ull << 32) || max_m * batch >= (1ull << 32)) return PEEL_EINVAL;
    if (ntrials == 0) return PEEL_OK;
    if (!sg_applicable(n, max_m, r, k))
        return sweep_union(n, r, k, m, seeds, ntrials, batch, out_rounds, out_core, workspace, ws_bytes, stream);
    const SGLayout L = sg_layout(n, max_m);
    if (ws_bytes < L.total) return PEEL_ENOMEM;
    std::vector<uint64_t> redo;
    peel_status st;
    {
        prof_begin_call();
        prof_hold(true);
        st = sweep_groups(n, r, k, m, seeds, ntrials, out_rounds, out_core, workspace, L, (cudaStream_t)stream, redo);
        prof_hold(false);
        prof_collect();
    }
    if (st != PEEL_OK || redo.empty()) return st;
    // trials whose count field overflowed: the union path (64-bit states), on the same workspace
    std::vector<uint64_t> rm(redo.size()), rs(redo.size()), rc(redo.size());
    std::vector<uint32_t> rr(redo.size());
    for (size_t i = 0; i < redo.size(); i++) { rm[i] = m[redo[i]]; rs[i] = seeds[redo[i]]; }
    st = sweep_union(n, r, k, rm.data(), rs.data(), redo.size(), batch, rr.data(), rc.data(), workspace, ws_bytes, stream);
    if (st != PEEL_OK) return st;
    for (size_t i = 0; i < redo.size(); i++) { out_rounds[redo[i]] = rr[i]; out_core[redo[i]] = rc[i]; }
    return PEEL_OK;
}
