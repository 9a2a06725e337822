// kcore.cu -- a2-a7: round-synchronous parallel peeling to the k-core on sm_100a.
//
// The method: round t removes the snapshot
// F_t = {alive v : deg_t(v) < k} and every alive edge with an endpoint in F_t;
// stop at the first empty F_t.  This file computes exactly that schedule with
// work proportional to the edges actually removed:
//
//  * build  -- per-vertex state from one coalesced pass over edges[m][r].
//              k <= 2 "packed": u64 word  (sum of incident edge ids mod 2^32) << 32 | count.
//              One 64-bit RED per endpoint adds (e << 32) + 1.  count lives in the low
//              half and never exceeds m < 2^32, so nothing carries into it; the id sum
//              wraps harmlessly in the high half.  When count == 1 the id sum IS the one
//              alive incident edge, so k = 2 needs no incidence lists.
//              k >= 3 "CSR": u32 degree histogram, exclusive scan, scatter of edge ids.
//  * rounds -- ONE cooperative persistent kernel runs every round, grid barrier between
//              rounds (the host is not involved; P:505-506's termination test is a device
//              counter).  Round 1: a scan of all n vertices for count < k.  Round t: every
//              alive edge of F_t is killed exactly once by test-and-clear of its alive bit
//              (atomicAnd returns the old word); the winner decrements the other endpoints;
//              the ONE decrement that takes a count from k to k-1 puts that vertex in
//              F_{t+1} -- no rescans, each vertex exactly once.
//              packed k = 2: a frontier ENTRY is (v, e) with e = v's one alive edge at the
//              start of round t+1, computed by the crossing decrement itself
//              (old id sum - killed edge): rounds >= 2 never re-read the state of a
//              frontier vertex.  If e dies in round t too, v's count reaches 0 and e's alive
//              bit is already clear at round t+1, so the entry does nothing -- exactly the
//              snapshot semantics.  Vertices with count 0 in F_t have nothing to kill and
//              get no entry; |F_t| is counted separately for survivors[t].
//  * output -- core_mask[v] = (count(v) >= k): a removed vertex had count < k when removed
//              and counts never increase.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "shard.h"

namespace peel {

static constexpr uint32_t STAT_CAP = 65536;  // per-round statistics kept on device
static constexpr int PEEL_BLOCK = 256;
static constexpr uint32_t SCAN_TILE = 2048;  // 256 threads x 8 elements

enum : uint32_t { ERR_BADVERTEX = 1u };

struct Ctl {
    ull nf[3];        // |F_t| (vertices removed in round t), rotating: round t uses nf[(t-1)%3]
    ull ne[3];        // frontier list lengths, same rotation
    ull rounds;       // number of non-empty rounds
    ull work;         // binned-round work-item counter
    uint32_t err;     // ERR_* bits
    uint32_t binovf;  // a vertex bin overflowed its capacity (binned build falls back)
    ull nlive[2];     // compacted rounds: live vertices after round t at nlive[t & 1] (build: [0])
    ull cwork;        // compacted rounds: the compaction pass's work-item counter (side stream)
};

// compacted rounds (kcompact.cuh): group records, per-bin live counts, A-item counters,
// per-edge-bin frontier regions and their counts
struct CompactLayout {
    size_t recs, live0, live1, adone, fecnt0, fecnt1, fe, rc;
    uint64_t enb, fe_stride;
};

struct Layout {
    size_t ctl, stats, sub, rtime, state, deg, off, bsum, adj, alive, F0, F1;
    size_t bins, bin_cursor, bin_base, bin_cap, entries;  // binned build (packed, n > BIN_MIN_N)
    size_t esort;                                          // binned rounds: edge-bin counters of the frontier sort
    uint64_t nbins, total_cap;
    bool compact;                                          // packed, n > BIN_MIN_N: kcompact.cuh's rounds
    CompactLayout cl;
    size_t total;
};

// Binned build: endpoint increments are partitioned into vertex bins of
// 2^BIN_SHIFT vertices (32 MB of state, L2-resident), then each bin is accumulated with
// L2 atomics and scanned for the round-1 frontier while it is still in L2.
static constexpr int BIN_SHIFT = 22;
static_assert(BIN_SHIFT == SHARD_BIN_SHIFT, "dist.cu stages decrements in kcore.cu's bins");
static constexpr uint64_t BIN_MIN_N = 1ull << 23;
// binned rounds sort the frontier by edge bin (2^EB_SHIFT edges: 512 KB of alive bits, 48 MB
// of r=3 rows) before the kill phase, so the blocks in flight test alive bits of one bin
static constexpr int EB_SHIFT = 22;  // below this the state fits L2: direct build

__host__ __device__ inline uint64_t bin_size(uint64_t n, uint64_t b) {
    uint64_t lo = b << BIN_SHIFT, hi = (b + 1) << BIN_SHIFT;
    return (hi < n ? hi : n) - lo;
}

// capacity of bin b: expected r m size/n plus 8 standard deviations plus 4096 (IEEE sqrt,
// identical on host and device); a bin that overflows sends the build down the direct path
// (a shard of nloc vertices of an n-vertex instance: its bins over [0, nloc), density r m / n)
__host__ __device__ inline uint64_t bin_capacity(uint64_t n, uint64_t nloc, uint64_t m, uint32_t r, uint64_t b) {
    uint64_t lam = (bin_size(nloc, b) * (uint64_t)r * m) / n;
    return lam + 8ull * (uint64_t)sqrt((double)lam) + 4096ull;
}

static inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static Layout layout(uint64_t n, uint64_t m, uint32_t r, bool csr) {
    Layout L;
    size_t o = 0;
    L.ctl = o; o += al(sizeof(Ctl));
    // per-round (|F_t|, killed_t) pairs right after the control block: one small copy brings
    // back the control block and the first STAT_HEAD rounds' statistics
    L.stats = o; o += al(2 * sizeof(ull) * (STAT_CAP + 1));
    L.sub = o; o += al(sizeof(ull) * 64);  // subround mode: per-class list counters
    L.rtime = o; o += al(sizeof(ull) * (STAT_CAP + 2));
    const size_t fe = csr ? sizeof(uint32_t) : sizeof(uint2);  // frontier element: v, or (v, e)
    if (!csr) {
        L.state = o; o += al(sizeof(ull) * n);
        L.deg = L.off = L.bsum = L.adj = 0;
    } else {
        L.state = 0;
        L.deg = o; o += al(sizeof(uint32_t) * n);
        L.off = o; o += al(sizeof(uint32_t) * n);
        L.bsum = o; o += al(sizeof(uint32_t) * ((n + SCAN_TILE - 1) / SCAN_TILE + 1));
        L.adj = o; o += al(sizeof(uint32_t) * r * m);
    }
    L.alive = o; o += al(sizeof(uint32_t) * ((m + 31) / 32));
    L.F0 = o; o += al(fe * n);
    L.F1 = o; o += al(fe * n);
    L.nbins = 0; L.total_cap = 0;
    L.bins = L.bin_cursor = L.bin_base = L.bin_cap = L.entries = 0;
    L.esort = 0;
    if (n > BIN_MIN_N) {  // packed: binned build + rounds; CSR: binned degree count + scatter
        L.nbins = (n + (1ull << BIN_SHIFT) - 1) >> BIN_SHIFT;
        for (uint64_t b = 0; b < L.nbins; b++) L.total_cap += bin_capacity(n, n, m, r, b);
        L.bins = o;
        L.bin_cursor = o; o += al(sizeof(ull) * L.nbins);
        L.bin_base = o; o += al(sizeof(ull) * L.nbins);
        L.bin_cap = o; o += al(sizeof(ull) * L.nbins);
        L.entries = o; o += al(sizeof(ull) * L.total_cap);
        L.esort = o; o += al(sizeof(ull) * 3 * (((m + (1ull << EB_SHIFT) - 1) >> EB_SHIFT) + 1));
    }
    L.compact = !csr && n > BIN_MIN_N;
    memset(&L.cl, 0, sizeof L.cl);
    if (L.compact) {
        CompactLayout &C = L.cl;
        C.enb = (m + (1ull << EB_SHIFT) - 1) >> EB_SHIFT;
        if (C.enb == 0) C.enb = 1;
        C.fe_stride = (uint64_t)r << EB_SHIFT;  // an edge bin's entries: <= r per edge (one per endpoint)
        C.recs = o; o += al(16 * ((n + 63) / 64));
        C.live0 = o; o += al(sizeof(ull) * L.nbins);
        C.live1 = o; o += al(sizeof(ull) * L.nbins);
        C.adone = o; o += al(sizeof(uint32_t) * 2 * L.nbins);  // dataflow build: zeroed / accumulated items per bin
        C.fecnt0 = o; o += al(sizeof(ull) * C.enb);
        C.fecnt1 = o; o += al(sizeof(ull) * C.enb);
        C.fe = o; o += al(sizeof(uint2) * C.enb * C.fe_stride);
        C.rc = o; o += al(64);  // RoundCtl
    }
    L.total = o;
    return L;
}

// ---------------------------------------------------------------------------
// build
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ bool load_edge(const uint32_t *__restrict__ edges, uint64_t e, uint64_t n,
                                          uint32_t (&u)[R]) {
    bool ok = true;
    #pragma unroll
    for (int j = 0; j < R; j++) {
        u[j] = __ldg(edges + e * R + j);
        ok &= (uint64_t)u[j] < n;
    }
    #pragma unroll
    for (int i = 0; i < R; i++)
        #pragma unroll
        for (int j = i + 1; j < R; j++) ok &= u[i] != u[j];
    return ok;
}

// packed k<=2 build: state[u] += (e << 32) + 1 for every endpoint (P:500-501's one-thread-
// per-item atomic update, applied to the count / id-sum accumulators); RED, no return.
template <int R>
__global__ void __launch_bounds__(256) build_packed_kernel(const uint32_t *__restrict__ edges,
                                                           uint64_t n, uint64_t m, ull *state,
                                                           Ctl *ctl) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u[R];
        if (!load_edge<R>(edges, e, n, u)) {
            atomicOr(&ctl->err, ERR_BADVERTEX);
            continue;
        }
        const ull inc = (e << 32) + 1ull;
        #pragma unroll
        for (int j = 0; j < R; j++) atomicAdd(state + u[j], inc);
    }
}

// ---- binned build ------------------------------------------------------------------------
__global__ void bin_init_kernel(uint64_t n, uint64_t nloc, uint64_t m, uint32_t r, uint64_t nbins, ull *cursor,
                                ull *base, ull *cap) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        ull o = 0;
        for (uint64_t b = 0; b < nbins; b++) {
            ull c = bin_capacity(n, nloc, m, r, b);
            cursor[b] = 0;
            base[b] = o;
            cap[b] = c;
            o += c;
        }
    }
}

static constexpr int PART_BLOCK = 256;
// 3072-entry chunks at 5 resident blocks per SM (43 registers, ~43 KB shared): C5 partition
// 12.6 -> 11.7 ms against 4096 entries at 4 blocks (62 registers); 2048 at 6 blocks: 12.3 ms
#ifndef PEEL_PART_ENTRIES
#define PEEL_PART_ENTRIES 3072
#endif
#ifndef PEEL_PART_MINB
#define PEEL_PART_MINB 5
#endif
static constexpr int PART_ENTRIES = PEEL_PART_ENTRIES;  // endpoint entries staged per chunk

// pass 1: partition the r m endpoint increments by vertex bin.  Per chunk of edges the
// block stages the chunk's edge words in shared memory with 16-byte coalesced loads,
// histograms bins in shared memory, reserves one contiguous run per bin with a single
// global atomic, counting-sorts the chunk's entries by bin in shared memory and writes
// them out so each bin's run is a coalesced store.  Stored entry =
// e << 32 | (u mod 2^BIN_SHIFT); in shared memory the full u is kept (bin = u >> BIN_SHIFT).
// Shared memory = 4 B + 8 B per entry + 20 B per bin + 1 B per edge (sized per launch).
template <int R>
__global__ void __launch_bounds__(PART_BLOCK, PEEL_PART_MINB) bin_partition_kernel(const uint32_t *__restrict__ edges,
                                                                      uint64_t n, uint64_t m, uint32_t nbins,
                                                                      ull *cursor, const ull *__restrict__ base,
                                                                      const ull *__restrict__ cap, ull *entries,
                                                                      uint32_t *err, uint32_t *binovf,
                                                                      uint64_t v0, uint64_t v1, uint64_t e0) {
    constexpr int CH = PART_ENTRIES / R;  // edges per chunk
    constexpr int CW = CH * R;            // edge words per chunk
    constexpr int CWP = (CW + 3) & ~3;    // padded: keeps every array below 16-byte aligned
    extern __shared__ unsigned char smem_raw[];
    ull *sent = (ull *)smem_raw;                  // [CWP]  (e << 32 | u), bin-sorted
    uint32_t *words = (uint32_t *)(sent + CWP);   // [CWP]  the chunk's edge words
    ull *gpos = (ull *)(words + CWP);             // [nbins]
    uint32_t *hist = (uint32_t *)(gpos + nbins);  // [nbins]
    uint32_t *offs = hist + nbins;                // [nbins]
    uint32_t *fill = offs + nbins;                // [nbins]
    __shared__ uint32_t total;
    const ull mask = (1ull << BIN_SHIFT) - 1;
    for (uint64_t c0 = e0 + (uint64_t)blockIdx.x * CH; c0 < m; c0 += (uint64_t)gridDim.x * CH) {  // edges [e0, m)
        const int ne = (int)min((uint64_t)CH, m - c0);
        const int nw = ne * R;
        for (uint32_t b = threadIdx.x; b < nbins; b += PART_BLOCK) hist[b] = 0;
        // stage the chunk's words (the chunk starts at word c0 R; 16-byte loads where aligned)
        const uint32_t *src = edges + c0 * R;
        if (threadIdx.x == 0) {  // the block's next chunk: into L2 while this one is sorted
            const uint64_t c1 = c0 + (uint64_t)gridDim.x * CH;
            if (c1 < m) {
                const uint64_t w1 = min((uint64_t)CW, (m - c1) * R);
                const uintptr_t p0 = (uintptr_t)(edges + c1 * R) & ~(uintptr_t)15;
                const uintptr_t p1 = ((uintptr_t)(edges + c1 * R + w1) + 15) & ~(uintptr_t)15;
                if (p1 > p0) prefetch_l2((const void *)p0, (uint32_t)(p1 - p0));
            }
        }
        if ((((uintptr_t)src) & 15) == 0) {
            const int nv = nw / 4;
            for (int i = threadIdx.x; i < nv; i += PART_BLOCK)
                reinterpret_cast<uint4 *>(words)[i] = __ldcs(reinterpret_cast<const uint4 *>(src) + i);
            for (int i = nv * 4 + threadIdx.x; i < nw; i += PART_BLOCK) words[i] = __ldcs(src + i);
        } else {
            for (int i = threadIdx.x; i < nw; i += PART_BLOCK) words[i] = __ldcs(src + i);
        }
        __syncthreads();
        // thread t takes edges t, t + 256, ...: validates each in registers, and ranks the
        // shard's endpoints [v0, v1) (local ids u - v0) in their bins with the histogram
        // atomic's return value; ids and ranks stay in registers for the scatter (round 2:
        // one pass over the staged words instead of a validation pass, a rank pass that
        // rewrote them and a scatter pass that re-read them)
        constexpr int EPT = (CH + PART_BLOCK - 1) / PART_BLOCK;  // edges per thread
        static_assert(EPT * R <= 32, "one keep bit per (edge, endpoint) of the thread");
        uint32_t lid[EPT][R], rank[EPT][R];
        uint32_t kept = 0;  // bit q R + j: lid[q][j] is kept (every u32 is a valid local id)
        #pragma unroll
        for (int q = 0; q < EPT; q++) {
            const int i = q * PART_BLOCK + threadIdx.x;
            if (i < ne) {
                uint32_t w[R];
                #pragma unroll
                for (int j = 0; j < R; j++) w[j] = words[i * R + j];
                bool ok = true;
                #pragma unroll
                for (int j = 0; j < R; j++) ok &= (uint64_t)w[j] < n;
                #pragma unroll
                for (int j = 0; j < R; j++)
                    #pragma unroll
                    for (int j2 = j + 1; j2 < R; j2++) ok &= w[j] != w[j2];
                if (!ok) atomicOr(err, ERR_BADVERTEX);
                #pragma unroll
                for (int j = 0; j < R; j++)
                    if (ok && (uint64_t)w[j] >= v0 && (uint64_t)w[j] < v1) {
                        lid[q][j] = (uint32_t)(w[j] - v0);
                        rank[q][j] = atomicAdd(&hist[lid[q][j] >> BIN_SHIFT], 1u);
                        kept |= 1u << (q * R + j);
                    }
            }
        }
        __syncthreads();
        // exclusive scan of hist over nbins (<= 1024): one warp
        if (threadIdx.x < 32) {
            const uint32_t per = (nbins + 31) / 32;
            uint32_t loc = 0;
            for (uint32_t q = 0; q < per; q++) {
                uint32_t b = threadIdx.x * per + q;
                loc += b < nbins ? hist[b] : 0;
            }
            uint32_t x = loc;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if ((int)threadIdx.x >= o) x += y;
            }
            uint32_t run = x - loc;
            for (uint32_t q = 0; q < per; q++) {
                uint32_t b = threadIdx.x * per + q;
                if (b < nbins) { offs[b] = run; run += hist[b]; }
            }
            if (threadIdx.x == 31) total = x;
        }
        __syncthreads();
        // gpos[b] <- the run's absolute start in the entry buffer, and fill[b] <- how many of
        // its entries still fit the bin (the write-out reads shared memory only)
        for (uint32_t b = threadIdx.x; b < nbins; b += PART_BLOCK)
            if (hist[b]) {
                const ull g = atomicAdd(cursor + b, (ull)hist[b]);
                const ull c = cap[b];
                if (g + hist[b] > c) atomicOr(binovf, 1u);
                gpos[b] = base[b] + g;
                fill[b] = (uint32_t)(g >= c ? 0ull : min((ull)hist[b], c - g));
            }
        #pragma unroll
        for (int q = 0; q < EPT; q++) {
            const uint64_t e = c0 + (uint64_t)(q * PART_BLOCK + threadIdx.x);
            #pragma unroll
            for (int j = 0; j < R; j++)
                if ((kept >> (q * R + j)) & 1u) sent[offs[lid[q][j] >> BIN_SHIFT] + rank[q][j]] = (e << 32) | lid[q][j];
        }
        __syncthreads();
        const uint32_t tot = total;
        for (uint32_t i = threadIdx.x; i < tot; i += PART_BLOCK) {
            const ull x = sent[i];
            const uint32_t b = (uint32_t)x >> BIN_SHIFT;
            const uint32_t q = i - offs[b];
            if (q < fill[b]) entries[gpos[b] + q] = x & ~(0xFFFFFFFFull ^ mask);
        }
        __syncthreads();
    }
}

static size_t partition_smem(int r, uint64_t nbins) {
    const size_t cw = (((size_t)(PART_ENTRIES / r) * r) + 3) & ~(size_t)3;
    return (sizeof(ull) + sizeof(uint32_t)) * cw + (sizeof(ull) + 3 * sizeof(uint32_t)) * nbins + PART_ENTRIES / r + 16;
}

// CSR build from the binned entries: blockIdx.y = bin, blocks scheduled bin-major, so the
// degree / offset range of the bin being processed (16 MB) stays L2-resident.
static constexpr int CSRB_PER = 16;  // entries per thread per block

__global__ void __launch_bounds__(256) csr_bin_deg_kernel(const ull *__restrict__ entries, const ull *__restrict__ base,
                                                          const ull *__restrict__ cursor, uint32_t *deg) {
    const uint32_t b = blockIdx.y;
    const ull cnt = cursor[b];
    const ull lo = (ull)blockIdx.x * 256 * CSRB_PER;
    if (lo >= cnt) return;
    const ull *ent = entries + base[b];
    uint32_t *d = deg + ((uint64_t)b << BIN_SHIFT);
    const ull mask = (1ull << BIN_SHIFT) - 1;
    #pragma unroll 4
    for (int i = 0; i < CSRB_PER; i++) {
        const ull p = lo + (ull)i * 256 + threadIdx.x;
        if (p < cnt) atomicAdd(d + (__ldcs(ent + p) & mask), 1u);
    }
}

// blockIdx.y = bin * 2^SUB_LOG + sub: each bin is scattered in 2^SUB_LOG passes over its
// entries, pass `sub` writing only the entries of its vertex sub-range, so the adjacency
// window being written (~r m 4 / (nbins 2^SUB_LOG) bytes) stays L2-resident
// (C4b: 1 pass 9.5 ms, 2 passes 7.0, 4 passes 7.8, 8 passes 12.2)
#ifndef PEEL_CSR_SUB_LOG
#define PEEL_CSR_SUB_LOG 1
#endif
static constexpr int CSR_SUB_LOG = PEEL_CSR_SUB_LOG;

__global__ void __launch_bounds__(256) csr_bin_scatter_kernel(const ull *__restrict__ entries, const ull *__restrict__ base,
                                                              const ull *__restrict__ cursor, uint32_t *off,
                                                              uint32_t *adj) {
    const uint32_t b = blockIdx.y >> CSR_SUB_LOG, sub = blockIdx.y & ((1u << CSR_SUB_LOG) - 1);
    const ull cnt = cursor[b];
    const ull lo = (ull)blockIdx.x * 256 * CSRB_PER;
    if (lo >= cnt) return;
    const ull *ent = entries + base[b];
    uint32_t *o = off + ((uint64_t)b << BIN_SHIFT);
    const ull mask = (1ull << BIN_SHIFT) - 1;
    #pragma unroll 4
    for (int i = 0; i < CSRB_PER; i++) {
        const ull p = lo + (ull)i * 256 + threadIdx.x;
        if (p < cnt) {
            const ull x = CSR_SUB_LOG ? __ldcg(ent + p) : __ldcs(ent + p);
            if ((uint32_t)((x & mask) >> (BIN_SHIFT - CSR_SUB_LOG)) == sub)
                adj[atomicAdd(o + (x & mask), 1u)] = (uint32_t)(x >> 32);
        }
    }
}

// binned build of a vertex shard (dist.cu): apply the bin-partitioned increments with 64-bit
// REDs, bin-major (blockIdx.y = bin), so each bin's 32 MB of state is L2-resident while applied
__global__ void __launch_bounds__(256) bin_red_kernel(const ull *__restrict__ entries, const ull *__restrict__ base,
                                                      const ull *__restrict__ cursor, ull *state) {
    const uint32_t b = blockIdx.y;
    const ull cnt = cursor[b];
    const ull lo = (ull)blockIdx.x * 256 * CSRB_PER;
    if (lo >= cnt) return;
    const ull *ent = entries + base[b];
    ull *st = state + ((uint64_t)b << BIN_SHIFT);
    const ull mask = (1ull << BIN_SHIFT) - 1;
    #pragma unroll 4
    for (int i = 0; i < CSRB_PER; i++) {
        const ull p = lo + (ull)i * 256 + threadIdx.x;
        if (p < cnt) {
            const ull x = __ldcs(ent + p);
            atomicAdd(st + (x & mask), (x & ~0xFFFFFFFFull) + 1ull);
        }
    }
}

// CSR build, pass 1: degree histogram
template <int R>
__global__ void __launch_bounds__(256) build_deg_kernel(const uint32_t *__restrict__ edges, uint64_t n,
                                                        uint64_t m, uint32_t *deg, Ctl *ctl) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u[R];
        if (!load_edge<R>(edges, e, n, u)) {
            atomicOr(&ctl->err, ERR_BADVERTEX);
            continue;
        }
        #pragma unroll
        for (int j = 0; j < R; j++) atomicAdd(deg + u[j], 1u);
    }
}

// exclusive scan of deg into off: tile pass (local exclusive scan + tile total)
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t ws[PEEL_BLOCK / 32];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < PEEL_BLOCK / 32 ? ws[lane] : 0;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < PEEL_BLOCK / 32) ws[lane] = s;
    }
    __syncthreads();
    uint32_t before = (w ? ws[w - 1] : 0) + x - v;
    *total = ws[PEEL_BLOCK / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(PEEL_BLOCK) scan_tiles_kernel(const uint32_t *__restrict__ deg,
                                                                uint64_t n, uint32_t *off,
                                                                uint32_t *bsum) {
    const int PER = SCAN_TILE / PEEL_BLOCK;
    uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * PER;
    uint32_t v[PER], s = 0;
    #pragma unroll
    for (int i = 0; i < PER; i++) {
        v[i] = base + i < n ? deg[base + i] : 0;
        s += v[i];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan(s, &tot);
    #pragma unroll
    for (int i = 0; i < PER; i++) {
        if (base + i < n) off[base + i] = ex;
        ex += v[i];
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(PEEL_BLOCK) scan_bsum_kernel(uint32_t *bsum, uint64_t nb) {
    uint32_t carry = 0;
    for (uint64_t b0 = 0; b0 < nb; b0 += PEEL_BLOCK) {
        uint64_t i = b0 + threadIdx.x;
        uint32_t v = i < nb ? bsum[i] : 0, tot;
        uint32_t ex = block_exclusive_scan(v, &tot);
        if (i < nb) bsum[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(PEEL_BLOCK) scan_add_kernel(uint32_t *off, uint64_t n,
                                                              const uint32_t *__restrict__ bsum) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        off[i] += bsum[i / SCAN_TILE];
}

// CSR build, pass 2: scatter edge ids; afterwards off[u] = END of u's list
template <int R>
__global__ void __launch_bounds__(256) scatter_kernel(const uint32_t *__restrict__ edges, uint64_t n,
                                                      uint64_t m, uint32_t *off, uint32_t *adj) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u[R];
        if (!load_edge<R>(edges, e, n, u)) continue;  // flagged by build_deg_kernel
        #pragma unroll
        for (int j = 0; j < R; j++) {
            uint32_t pos = atomicAdd(off + u[j], 1u);
            adj[pos] = (uint32_t)e;
        }
    }
}

// block-aggregated append queues (common.cuh): one global atomic per block iteration
static constexpr int U = 4;                      // frontier entries per thread per iteration (MLP)
static constexpr int CHUNK = PEEL_BLOCK * U;     // entries per block iteration
static constexpr int QCAP = 2 * CHUNK;
template <typename T>
using BlockQueue = BlockQueueT<T, QCAP, PEEL_BLOCK>;

// ---------------------------------------------------------------------------
// the round loop: one cooperative persistent kernel
// ---------------------------------------------------------------------------
struct PeelArgs {
    const uint32_t *edges;
    uint64_t n, m;
    uint32_t k;
    uint32_t stat_cap;
    ull *state;              // packed path
    uint32_t *deg;           // CSR path
    const uint32_t *off_end; // CSR path: end of u's adjacency list
    const uint32_t *adj;     // CSR path
    uint32_t *alive;
    void *F[2];              // packed: uint2 (v, e) entries; CSR: u32 vertices
    Ctl *ctl;
    ull *stats;              // [2 t] = |F_{t+1}|, [2 t + 1] = edges killed in round t+1
    uint8_t *core_mask;
    uint32_t *peel_round;
    int mask_vec;            // core_mask is 16-byte aligned
    int edges_vec;           // edges is 16-byte aligned (vector row loads)
    int f1_ready;            // packed: F_1 was emitted by the binned build
    uint32_t t0;             // first round run by the persistent kernel (earlier rounds were binned)
    uint32_t r;              // subround mode: number of vertex classes (= r)
    uint64_t cs;             // subround mode: class size n / r
    ull *sub;                // subround mode: counters [class][buffer][kind: 0 |F|, 1 entries]
    ull *rtime;              // %globaltimer at the start of each round (profiling)
    uint64_t v0;             // vertex id of state[0] (a shard of dist.cu; 0 otherwise)
};

__device__ __forceinline__ uint32_t count_of(ull w) { return (uint32_t)w; }
__device__ __forceinline__ uint32_t idsum_of(ull w) { return (uint32_t)(w >> 32); }

template <bool CSR>
__device__ void write_core_mask(const PeelArgs &a, uint64_t tid, uint64_t nthr) {
    // core_mask[v] = count(v) >= k (counts only decrease).  Warp-coalesced: each thread turns
    // one 16-byte load (2 packed states / 4 CSR degrees) into one 2- / 4-byte mask store, so a
    // warp instruction moves 512 B of state and 64 / 128 B of mask; UM loads are issued before
    // any store so enough bytes are in flight to stream at HBM rate.
    constexpr int UM = 4;
    constexpr uint64_t VPL = CSR ? 4 : 2;  // vertices per 16-byte load
    const uint32_t k = a.k;
    const uint4 *src = CSR ? reinterpret_cast<const uint4 *>(a.deg) : reinterpret_cast<const uint4 *>(a.state);
    const uint64_t nv = (a.mask_vec && ((uintptr_t)src & 15) == 0) ? a.n / VPL : 0;  // whole 16-byte groups
    for (uint64_t w0 = tid; w0 < nv; w0 += UM * nthr) {
        uint4 x[UM];
        #pragma unroll
        for (int j = 0; j < UM; j++) {
            const uint64_t w = w0 + j * nthr;
            x[j] = w < nv ? __ldcs(src + w) : make_uint4(0u, 0u, 0u, 0u);
        }
        #pragma unroll
        for (int j = 0; j < UM; j++) {
            const uint64_t w = w0 + j * nthr;
            if (w >= nv) break;
            if (CSR) {
                const uint32_t b = (uint32_t)(x[j].x >= k) | (uint32_t)(x[j].y >= k) << 8 |
                                   (uint32_t)(x[j].z >= k) << 16 | (uint32_t)(x[j].w >= k) << 24;
                reinterpret_cast<uint32_t *>(a.core_mask)[w] = b;
            } else {  // packed state: the count is the low 32-bit word of each u64
                const uint16_t b = (uint16_t)((x[j].x >= k) | (x[j].z >= k) << 8);
                reinterpret_cast<uint16_t *>(a.core_mask)[w] = b;
            }
        }
    }
    for (uint64_t v = nv * VPL + tid; v < a.n; v += nthr) {
        uint32_t c = CSR ? ld_cg_u32(a.deg + v) : count_of(ld_cg_u64(a.state + v));
        a.core_mask[v] = c >= k ? 1 : 0;
    }
}

// Round-1 frontier over vertices [lo, hi): F_1 = {v : count(v) < k}; a vertex with
// count 1 gets the entry (v, its one edge = the id sum).  Block-uniform: every
// thread of the block must call it with the same range.
__device__ __forceinline__ void scan_emit(const PeelArgs &a, BlockQueue<uint2> &q, int &slot, uint64_t lo,
                                          uint64_t hi, ull &removed) {
    uint2 *F = (uint2 *)a.F[0];
    ull *cnt = &a.ctl->ne[0];
    for (uint64_t base = lo + (uint64_t)blockIdx.x * CHUNK; base < hi; base += (uint64_t)gridDim.x * CHUNK) {
        ull w[U];
        #pragma unroll
        for (int j = 0; j < U; j++) {
            const uint64_t v = base + (uint64_t)j * PEEL_BLOCK + threadIdx.x;
            w[j] = v < hi ? ld_cg_u64(a.state + v) : ~0ull;
        }
        #pragma unroll
        for (int j = 0; j < U; j++) {
            const uint64_t v = base + (uint64_t)j * PEEL_BLOCK + threadIdx.x;
            if (v < hi && count_of(w[j]) < a.k) {
                removed++;
                if (a.peel_round) a.peel_round[v] = 1;
                if (count_of(w[j]) == 1)  // k = 2: its one edge is the id sum
                    bq_push(q, slot, make_uint2((uint32_t)v, idsum_of(w[j])), F, cnt);
            }
        }
        bq_flush(q, slot, F, cnt);
        slot ^= 1;
    }
}

// pass 2 of the binned build (cooperative): for each bin b in order, zero its 32 MB of
// state, grid barrier, apply its entries with L2-resident 64-bit REDs, grid barrier,
// then (overlapped with zeroing bin b+1) scan it for the round-1 frontier while it is
// still in L2.  If any bin overflowed in pass 1, fall back to the direct build.
struct BinArgs {
    uint64_t nbins;
    const ull *cursor, *base, *cap, *entries;
};

template <int R>
// 6 resident blocks per SM (40 registers): C5 18.7 -> 18.5 ms against the compiler's 48
// registers (5 blocks)
__global__ void __launch_bounds__(PEEL_BLOCK, 6) bin_accumulate_kernel(PeelArgs a, BinArgs bn) {
    cg::grid_group grid = cg::this_grid();
    __shared__ BlockQueue<uint2> q;
    Ctl *ctl = a.ctl;
    if (ld_cg_u32(&ctl->err) & ERR_BADVERTEX) return;
    bq_init(q);
    __syncthreads();
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    int slot = 0;
    ull removed = 0;
    if (ld_cg_u32(&ctl->binovf)) {
        for (uint64_t v = tid; v < a.n; v += nthr) a.state[v] = 0ull;
        grid.sync();
        for (uint64_t e = tid; e < a.m; e += nthr) {
            uint32_t u[R];
            if (!load_edge<R>(a.edges, e, a.n, u)) continue;
            const ull inc = (e << 32) + 1ull;
            #pragma unroll
            for (int j = 0; j < R; j++) atomicAdd(a.state + u[j], inc);
        }
        grid.sync();
        scan_emit(a, q, slot, 0, a.n, removed);
    } else {
        const ull mask = (1ull << BIN_SHIFT) - 1;
        for (uint64_t b = 0; b <= bn.nbins; b++) {
            if (b > 0) {
                const uint64_t lo = (b - 1) << BIN_SHIFT;
                scan_emit(a, q, slot, lo, lo + bin_size(a.n, b - 1), removed);
            }
            if (b < bn.nbins) {
                const uint64_t lo = b << BIN_SHIFT, sz = bin_size(a.n, b);
                ulonglong2 *z = reinterpret_cast<ulonglong2 *>(a.state + lo);  // lo is 2^22-aligned
                for (uint64_t i = tid; i < sz / 2; i += nthr) z[i] = make_ulonglong2(0ull, 0ull);
                if ((sz & 1) && tid == 0) a.state[lo + sz - 1] = 0ull;
            }
            grid.sync();
            if (b < bn.nbins) {
                ull *st = a.state + (b << BIN_SHIFT);
                const ull *ent = bn.entries + bn.base[b];
                const ull cnt = min(bn.cursor[b], bn.cap[b]);
                for (ull i = tid; i < cnt; i += nthr) {
                    const ull x = __ldcs(ent + i);
                    atomicAdd(st + (x & mask), (x & ~0xFFFFFFFFull) + 1ull);
                }
            }
            grid.sync();
        }
    }
    block_add<PEEL_BLOCK>(&ctl->nf[0], removed);
}

// ---- binned rounds (large frontiers) --------------------------------------------------------
// A round whose frontier is a large fraction of n touches most 64 B granules of the state,
// so applying its decrements as random DRAM read-modify-writes (~20 G/s on B200) loses to
// streaming: phase K kills edges and partitions the decrements (e << 32 | u) by vertex bin,
// reusing the build's entry buffer (a round's decrements of bin b are a subset of the build's
// entries of bin b, so capacities always suffice); phase D applies them bin-major with
// L2-resident returning atomics while the next bin's state is prefetched into L2.  The
// crossing rule (old count == k) and the (v, e) frontier entries are those of the persistent
// kernel, so the schedule is unchanged.
// 3 entries per thread at 5 resident blocks per SM (48 registers): C5 kill 24.4-24.8 ->
// 24.0 ms against 4 at 4 blocks (62 registers); 2 at 6 blocks: 27.6 ms
#ifndef PEEL_KU
#define PEEL_KU 3
#endif
#ifndef PEEL_KILL_MINB
#define PEEL_KILL_MINB 5
#endif
static constexpr int KU = PEEL_KU;                 // frontier entries per thread per K iteration
static constexpr int KCH = PART_BLOCK * KU;       // entries per block iteration
#ifndef PEEL_DCH
#define PEEL_DCH 512
#endif
static constexpr int DCH = PEEL_DCH;                  // decrement entries per D work item (in-flight window ~ one bin)

struct BinRound {
    uint32_t nbins;
    ull *cursor;
    const ull *base;
    ull *entries;
    ull *work;          // D work-item counter
    uint32_t t;         // the round
    const uint2 *Fsrc;  // K: the round's frontier entries (edge-sorted copy), or null: F[(t-1)&1]
    ull *ehist;         // D: histogram of F_{t+1} by edge bin for the next round's sort, or null
    uint32_t enb;       // D: edge bins
};

template <int R>
__global__ void __launch_bounds__(PART_BLOCK, PEEL_KILL_MINB) round_kill_partition_kernel(PeelArgs a, BinRound br) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t nbins = br.nbins;
    ull *sorted = (ull *)smem_raw;                       // [(R-1) KCH] the chunk's decrements, bin-sorted
    ull *gpos = sorted + (R - 1) * KCH;                  // [nbins]
    uint32_t *hist = (uint32_t *)(gpos + nbins);         // [nbins]
    uint32_t *offs = hist + nbins;                       // [nbins]
    __shared__ uint32_t total;
    Ctl *ctl = a.ctl;
    const uint32_t t = br.t;
    const ull nE = ld_cg_u64(&ctl->ne[(t - 1) % 3]);
    const uint2 *Fc = br.Fsrc ? br.Fsrc : (const uint2 *)a.F[(t - 1) & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
        a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap)] = ld_cg_u64(&ctl->nf[(t - 1) % 3]);
        ctl->nf[(t + 1) % 3] = 0;
        ctl->ne[(t + 1) % 3] = 0;
    }
    const ull mask = (1ull << BIN_SHIFT) - 1;
    ull kills = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * KCH; base < nE; base += (uint64_t)gridDim.x * KCH) {
        for (uint32_t b = threadIdx.x; b < nbins; b += PART_BLOCK) hist[b] = 0;
        uint2 ent[KU];
        bool win[KU];
        #pragma unroll
        for (int j = 0; j < KU; j++) {
            const uint64_t i = base + (uint64_t)j * PART_BLOCK + threadIdx.x;
            ent[j] = i < nE ? __ldcg(Fc + i) : make_uint2(0u, 0u);
        }
        #pragma unroll
        for (int j = 0; j < KU; j++) {
            const uint64_t i = base + (uint64_t)j * PART_BLOCK + threadIdx.x;
            win[j] = false;
            if (i < nE) {
                const uint32_t e = ent[j].y, bit = 1u << (e & 31);
                win[j] = (atomicAnd(a.alive + (e >> 5), ~bit) & bit) != 0;
            }
        }
        uint32_t ue[KU][R];
        #pragma unroll
        for (int j = 0; j < KU; j++)
            if (win[j]) {
                kills++;
                load_row<R>(a.edges, ent[j].y, a.m, a.edges_vec, ue[j]);
            }
        __syncthreads();  // hist zeroed
        // the histogram atomic's return value is the decrement's rank within its bin: the
        // decrements stay in registers until the bin offsets are known (no unsorted copy)
        uint32_t rk[KU][R];
        #pragma unroll
        for (int j = 0; j < KU; j++)
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (win[j] && ue[j][r] != ent[j].x) rk[j][r] = atomicAdd(&hist[ue[j][r] >> BIN_SHIFT], 1u);
        __syncthreads();
        if (threadIdx.x < 32) {  // exclusive scan of hist over the bins: one warp
            const uint32_t per = (nbins + 31) / 32;
            uint32_t loc = 0;
            for (uint32_t q2 = 0; q2 < per; q2++) {
                uint32_t b = threadIdx.x * per + q2;
                loc += b < nbins ? hist[b] : 0;
            }
            uint32_t z = loc;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
                if (threadIdx.x >= (unsigned)o) z += y;
            }
            uint32_t run = z - loc;
            for (uint32_t q2 = 0; q2 < per; q2++) {
                uint32_t b = threadIdx.x * per + q2;
                if (b < nbins) { offs[b] = run; run += hist[b]; }
            }
            if (threadIdx.x == 31) total = z;
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nbins; b += PART_BLOCK)
            if (hist[b]) gpos[b] = atomicAdd(br.cursor + b, (ull)hist[b]);
        #pragma unroll
        for (int j = 0; j < KU; j++)
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (win[j] && ue[j][r] != ent[j].x)
                    sorted[offs[ue[j][r] >> BIN_SHIFT] + rk[j][r]] = ((ull)ent[j].y << 32) | ue[j][r];
        __syncthreads();
        const uint32_t tot = total;
        for (uint32_t i = threadIdx.x; i < tot; i += PART_BLOCK) {
            const ull v = sorted[i];
            const uint32_t b = (uint32_t)v >> BIN_SHIFT;
            br.entries[br.base[b] + gpos[b] + (i - offs[b])] = v & ~(0xFFFFFFFFull ^ mask);
        }
        __syncthreads();
    }
    block_add<PART_BLOCK>(&a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap) + 1], kills);
}

// ---- frontier sort by edge bin (binned rounds) ---------------------------------------------
// Two-pass counting sort of the entries (v, e) by e >> EB_SHIFT: per-block shared histograms,
// one scan, then a scatter in which each block counting-sorts a chunk in shared memory and
// writes one run per bin.  The kill phase then reads the entries in edge-bin order, so the
// alive bits (and the rows) it touches at a time cover ~one edge bin: L2 hits instead of
// random DRAM granules.
#ifndef PEEL_ES_CH
#define PEEL_ES_CH 4096
#endif
static constexpr int ES_CH = PEEL_ES_CH;  // entries per chunk (scatter)
// 5 resident scatter blocks per SM (48 registers) and a grid of 5 per SM: C5 sort 5.6 -> 5.25
// ms; 4 blocks at 64 registers 5.6, 6 at 40 (spilling) 5.3, 8 per SM 6.5 ms
static constexpr int ES_BLOCKS = 5;

__global__ void __launch_bounds__(256) esort_hist_kernel(const uint2 *__restrict__ F, const ull *__restrict__ pN,
                                                         uint32_t nb, ull *ghist) {
    extern __shared__ uint32_t sh[];
    for (uint32_t b = threadIdx.x; b < nb; b += 256) sh[b] = 0;
    __syncthreads();
    const ull N = ld_cg_u64(pN);
    for (ull i = blockIdx.x * 256ull + threadIdx.x; i < N; i += (ull)gridDim.x * 256)
        atomicAdd(&sh[__ldcg(&F[i].y) >> EB_SHIFT], 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += 256)
        if (sh[b]) atomicAdd(ghist + b, (ull)sh[b]);
}

// ghist: the entries per edge bin (complete before the launch); cursor: zeroed.  Every block
// derives the bins' start offsets from ghist itself (no separate scan launch).
__global__ void __launch_bounds__(256, ES_BLOCKS) esort_scatter_kernel(const uint2 *__restrict__ F, const ull *__restrict__ pN,
                                                            uint32_t nb, const ull *__restrict__ ghist, ull *cursor,
                                                            uint2 *out) {
    extern __shared__ unsigned char smem_raw[];
    uint2 *buf = (uint2 *)smem_raw;              // [ES_CH] the chunk, bin-sorted
    ull *gpos = (ull *)(buf + ES_CH);            // [nb]
    ull *gstart = gpos + nb;                     // [nb] exclusive prefix of ghist
    uint32_t *hist = (uint32_t *)(gstart + nb);  // [nb]
    uint32_t *offs = hist + nb;                  // [nb]
    uint32_t *fill = offs + nb;                  // [nb]
    if (threadIdx.x < 32) {
        const uint32_t per = (nb + 31) / 32;
        ull loc = 0;
        for (uint32_t q = 0; q < per; q++) {
            const uint32_t b = threadIdx.x * per + q;
            loc += b < nb ? ghist[b] : 0;
        }
        ull x = loc;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const ull y = __shfl_up_sync(0xffffffffu, x, o);
            if ((int)threadIdx.x >= o) x += y;
        }
        ull run = x - loc;
        for (uint32_t q = 0; q < per; q++) {
            const uint32_t b = threadIdx.x * per + q;
            if (b < nb) { gstart[b] = run; run += ghist[b]; }
        }
    }
    __syncthreads();
    const ull N = ld_cg_u64(pN);
    for (ull c0 = (ull)blockIdx.x * ES_CH; c0 < N; c0 += (ull)gridDim.x * ES_CH) {
        const uint32_t ne = (uint32_t)min((ull)ES_CH, N - c0);
        for (uint32_t b = threadIdx.x; b < nb; b += 256) { hist[b] = 0; fill[b] = 0; }
        __syncthreads();
        uint2 v[ES_CH / 256];
        #pragma unroll
        for (int j = 0; j < ES_CH / 256; j++) {
            const uint32_t i = j * 256 + threadIdx.x;
            v[j] = i < ne ? __ldcs(F + c0 + i) : make_uint2(0u, 0u);
            if (i < ne) atomicAdd(&hist[v[j].y >> EB_SHIFT], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // exclusive scan of hist (nb <= 1024): one warp
            const uint32_t per = (nb + 31) / 32;
            uint32_t loc = 0;
            for (uint32_t q = 0; q < per; q++) {
                const uint32_t b = threadIdx.x * per + q;
                loc += b < nb ? hist[b] : 0;
            }
            uint32_t x = loc;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if ((int)threadIdx.x >= o) x += y;
            }
            uint32_t run = x - loc;
            for (uint32_t q = 0; q < per; q++) {
                const uint32_t b = threadIdx.x * per + q;
                if (b < nb) { offs[b] = run; run += hist[b]; }
            }
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += 256)
            if (hist[b]) gpos[b] = gstart[b] + atomicAdd(cursor + b, (ull)hist[b]);
        #pragma unroll
        for (int j = 0; j < ES_CH / 256; j++) {
            const uint32_t i = j * 256 + threadIdx.x;
            if (i < ne) {
                const uint32_t b = v[j].y >> EB_SHIFT;
                buf[offs[b] + atomicAdd(&fill[b], 1u)] = v[j];
            }
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < ne; i += 256) {
            const uint2 x = buf[i];
            const uint32_t b = x.y >> EB_SHIFT;
            out[gpos[b] + (i - offs[b])] = x;
        }
        __syncthreads();
    }
}

static size_t esort_scatter_smem(uint32_t nb) {
    return sizeof(uint2) * ES_CH + (2 * sizeof(ull) + 3 * sizeof(uint32_t)) * nb;
}

static size_t kill_partition_smem(int r, uint32_t nbins) {
    return sizeof(ull) * (size_t)(r - 1) * KCH + (sizeof(ull) + 2 * sizeof(uint32_t)) * nbins;
}


// phase D: apply the round's decrements bin-major; work items of DCH entries are taken in
// bin order from a global counter, so the blocks in flight share one or two bins (L2-resident).
// a small crossing queue (<= DCH / PEEL_BLOCK pushes per thread per work item; overflow
// falls back to global appends): less shared memory, more resident blocks, more atomics in flight
typedef BlockQueueT<uint2, 2 * PEEL_BLOCK, PEEL_BLOCK> ApplyQ;

__global__ void __launch_bounds__(PEEL_BLOCK) round_apply_kernel(PeelArgs a, BinRound br) {
    extern __shared__ unsigned char smem_raw[];
    uint32_t *pre = (uint32_t *)smem_raw;  // [nbins + 1] prefix of work items per bin
    uint32_t *ehs = pre + br.nbins + 1;    // [enb] F_{t+1} by edge bin (when br.ehist)
    __shared__ ApplyQ q;
    __shared__ ull item;
    Ctl *ctl = a.ctl;
    const uint32_t t = br.t, nbins = br.nbins, k = a.k;
    if (br.ehist)
        for (uint32_t b = threadIdx.x; b < br.enb; b += PEEL_BLOCK) ehs[b] = 0;
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t b = 0; b < nbins; b++) {
            pre[b] = acc;
            acc += (uint32_t)((ld_cg_u64(br.cursor + b) + DCH - 1) / DCH);
        }
        pre[nbins] = acc;
    }
    bq_init(q);
    __syncthreads();
    const uint32_t nitems = pre[nbins];
    uint2 *Fn = (uint2 *)a.F[t & 1];
    ull *cn = &ctl->ne[t % 3];
    const ull mask = (1ull << BIN_SHIFT) - 1;
    ull crossed = 0;
    int slot = 0;
    for (;;) {
        if (threadIdx.x == 0) item = atomicAdd(br.work, 1ull);
        __syncthreads();
        const ull c = item;
        if (c >= nitems) break;
        uint32_t lo = 0, hi = nbins;  // bin b with pre[b] <= c < pre[b+1]
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= c) lo = mid; else hi = mid;
        }
        const uint32_t b = lo, j = (uint32_t)c - pre[b];
        if (threadIdx.x == 0 && b + 1 < nbins) {
            // prefetch slice j of the next bin's state (its items follow this bin's)
            const uint32_t nj = pre[b + 1] - pre[b];
            const uint64_t bytes = bin_size(a.n, b + 1) * sizeof(ull);
            const uint64_t sl = ((bytes + nj - 1) / nj + 15) & ~15ull;
            const uint64_t off = (uint64_t)j * sl;
            if (off < bytes) {
                const uint32_t len = (uint32_t)min((ull)sl, (ull)((bytes - off + 15) & ~15ull));
                prefetch_l2((const char *)(a.state + ((uint64_t)(b + 1) << BIN_SHIFT)) + off, len);
            }
        }
        const ull cnt = ld_cg_u64(br.cursor + b);
        const ull *ent = br.entries + br.base[b] + (ull)j * DCH;
        const uint32_t nin = (uint32_t)min((ull)DCH, cnt - (ull)j * DCH);
        ull *st = a.state + ((uint64_t)b << BIN_SHIFT);
        // all DU entries of a thread are loaded and their returning atomics issued before any
        // result is used: DU atomics in flight per thread
        constexpr int DU = DCH / PEEL_BLOCK;
        ull x[DU], old[DU];
        #pragma unroll
        for (int r = 0; r < DU; r++) {
            const uint32_t i = threadIdx.x + r * PEEL_BLOCK;
            x[r] = i < nin ? __ldcs(ent + i) : 0ull;
        }
        #pragma unroll
        for (int r = 0; r < DU; r++) {
            const uint32_t i = threadIdx.x + r * PEEL_BLOCK;
            old[r] = 0;
            if (i < nin) old[r] = atomicAdd(st + (x[r] & mask), 0ull - ((x[r] & ~0xFFFFFFFFull) + 1ull));
        }
        #pragma unroll
        for (int r = 0; r < DU; r++) {
            const uint32_t i = threadIdx.x + r * PEEL_BLOCK;
            if (i < nin && count_of(old[r]) == k) {
                crossed++;
                const uint32_t u = (uint32_t)(a.v0 + (b << BIN_SHIFT)) + (uint32_t)(x[r] & mask);
                const uint32_t e2 = idsum_of(old[r]) - (uint32_t)(x[r] >> 32);
                if (a.peel_round) a.peel_round[u] = t + 1;
                if (br.ehist) atomicAdd(&ehs[e2 >> EB_SHIFT], 1u);
                bq_push(q, slot, make_uint2(u, e2), Fn, cn);
            }
        }
        bq_flush(q, slot, Fn, cn);
        slot ^= 1;
        __syncthreads();  // item is rewritten next iteration
    }
    if (br.ehist) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < br.enb; b += PEEL_BLOCK)
            if (ehs[b]) atomicAdd(br.ehist + b, (ull)ehs[b]);
    }
    block_add<PEEL_BLOCK>(&ctl->nf[t % 3], crossed);
}

// ---- small instances: the whole peel in ONE thread-block cluster's distributed shared memory
// A round of the cooperative kernel is a chain of ~8 dependent global-memory operations plus
// a grid barrier: ~11 us at n = 10^5 whatever the grid size (measured with per-phase clock64
// traces).  For n up to ~1.4e5 every per-vertex and per-edge word fits the
// shared memory of a 16-CTA cluster, so the chain runs on DSMEM (cross-CTA ~215 cycles,
// local ~38) and the rounds are separated by the hardware cluster barrier:
//   CTA c owns vertices [c nl, (c+1) nl)  -> its packed states (count | id sum << 32) and the
//        frontier lists of those vertices (each vertex joins a frontier once: capacity nl);
//   round t: each CTA walks its own list L_t; an entry (u, e) test-and-clears e's alive bit
//        (global bitmap, L2-resident; exactly-once kill), reads e's row (L2-resident), and
//        decrements every other endpoint w in w's owner CTA; a k -> k-1 crossing appends
//        (w, id sum - e) to the owner's L_{t+1}.  Per-round totals meet in CTA 0.
// Same schedule, statistics and outputs as peel_packed_kernel (the state is built by
// build_packed_kernel in global memory first and copied in).
static constexpr int CL_THREADS = 1024;
static constexpr int CL_MAX = 16;

struct ClusterShape {
    uint32_t cs;      // CTAs in the cluster
    uint32_t nl;      // vertices per CTA (the last may have fewer)
    size_t smem;      // dynamic shared memory per CTA
};

static ClusterShape cluster_shape(uint64_t n, uint64_t m, uint32_t cs) {
    ClusterShape c;
    c.cs = cs;
    c.nl = (uint32_t)((n + cs - 1) / cs);
    (void)m;
    c.smem = (size_t)c.nl * (sizeof(ull) + 2 * sizeof(uint2));
    return c;
}

template <int R>
__global__ void __launch_bounds__(CL_THREADS, 1) peel_cluster_kernel(PeelArgs a, ClusterShape cs) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t c = cluster.block_rank();
    const uint32_t nl = cs.nl;
    ull *st = (ull *)smem_raw;                            // [nl] packed states of owned vertices
    uint2 *L0 = (uint2 *)(st + nl);                       // [nl] frontier list, round parity 0
    uint2 *L1 = L0 + nl;                                  // [nl] parity 1
    __shared__ uint32_t fcnt[3];                          // list lengths, round t appends fcnt[t % 3]
    __shared__ ull red[3][2];                             // CTA 0: (crossings, kills) of round t at [t % 3]
    __shared__ ull wred[CL_THREADS / 32][2];
    const uint32_t tid = threadIdx.x;
    const uint32_t k = a.k;
    const uint64_t v0 = (uint64_t)c * nl;
    const uint32_t nown = v0 >= a.n ? 0u : (uint32_t)min((uint64_t)nl, a.n - v0);
    if (ld_cg_u32(&a.ctl->err) & ERR_BADVERTEX) return;  // uniform over the cluster

    // block reduction of two counters, then one DSMEM atomic pair into CTA 0's red[slot]
    auto reduce_to_cta0 = [&](ull x, ull y, uint32_t slot) {
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            x += __shfl_down_sync(0xffffffffu, x, o);
            y += __shfl_down_sync(0xffffffffu, y, o);
        }
        if ((tid & 31) == 0) { wred[tid >> 5][0] = x; wred[tid >> 5][1] = y; }
        __syncthreads();
        if (tid < 32) {
            x = wred[tid][0];
            y = wred[tid][1];
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                x += __shfl_down_sync(0xffffffffu, x, o);
                y += __shfl_down_sync(0xffffffffu, y, o);
            }
            if (tid == 0) {
                ull *r0 = cluster.map_shared_rank(&red[slot][0], 0);
                if (x) atomicAdd(r0, x);
                if (y) atomicAdd(r0 + 1, y);
            }
        }
    };

    // ---- load: owned states, all alive bits set, counters zero; round-1 frontier ----
    for (uint32_t i = tid; i < nown; i += CL_THREADS) st[i] = ld_cg_u64(a.state + v0 + i);
    if (tid < 3) {
        fcnt[tid] = 0;
        red[tid][0] = red[tid][1] = 0;
    }
    cluster.sync();  // every CTA initialised before any DSMEM access (the alive bits were set by the host)
    ull removed = 0;
    for (uint32_t i = tid; i < nown; i += CL_THREADS) {
        const ull w = st[i];
        if (count_of(w) < k) {
            removed++;
            if (a.peel_round) a.peel_round[v0 + i] = 1;
            if (count_of(w) == 1) L0[atomicAdd(&fcnt[0], 1u)] = make_uint2((uint32_t)(v0 + i), idsum_of(w));
        }
    }
    reduce_to_cta0(removed, 0, 0);
    cluster.sync();
    ull nF = *cluster.map_shared_rank(&red[0][0], 0);  // |F_1|; red[0] is zeroed after B_1

    uint32_t t = 1;
    while (nF != 0) {
        if (c == 0 && tid == 0) {
            if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
            a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap)] = nF;
        }
        const uint2 *Lc = (t & 1) ? L0 : L1;              // L_t lives in L[(t-1) & 1]
        const uint32_t nE = fcnt[(t - 1) % 3];
        const uint32_t nslot = t % 3;                     // L_{t+1}'s counter
        const uint32_t nlist = t & 1;                     // L_{t+1}'s array
        ull kills = 0, crossed = 0;
        for (uint32_t i = tid; i < nE; i += CL_THREADS) {
            const uint2 ent = Lc[i];
            const uint32_t e = ent.y;
            // exactly-once kill on the global alive bitmap: L2 atomics beat DSMEM atomics here
            // (C1 round loop 87 -> 78 us with the bits in the owner CTAs' shared memory)
            const uint32_t bit = 1u << (e & 31);
            if (!(atomicAnd(a.alive + (e >> 5), ~bit) & bit)) continue;
            kills++;
            uint32_t row[R];
            load_row<R>(a.edges, e, a.m, a.edges_vec, row);
            const ull dec = 0ull - (((ull)e << 32) + 1ull);
            ull old[R];
            #pragma unroll
            for (int r = 0; r < R; r++) {
                old[r] = ~0ull;
                if (row[r] != ent.x) {
                    const uint32_t ow = row[r] / nl;
                    old[r] = atomicAdd(cluster.map_shared_rank(st + (row[r] - ow * nl), ow), dec);
                }
            }
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (count_of(old[r]) == k) {                // k -> k-1: row[r] joins F_{t+1}
                    crossed++;
                    const uint32_t w = row[r], ow = w / nl;
                    if (a.peel_round) a.peel_round[w] = t + 1;
                    const uint32_t pos = atomicAdd(cluster.map_shared_rank(&fcnt[nslot], ow), 1u);
                    uint2 *dst = cluster.map_shared_rank((nlist ? L1 : L0) + pos, ow);
                    *dst = make_uint2(w, idsum_of(old[r]) - e);
                }
        }
        reduce_to_cta0(crossed, kills, t % 3);
        cluster.sync();                                   // B_t: round t complete everywhere
        const ull *r0 = cluster.map_shared_rank(&red[t % 3][0], 0);
        nF = r0[0];
        if (c == 0 && tid == 0) {
            a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap) + 1] = r0[1];
            red[(t + 2) % 3][0] = red[(t + 2) % 3][1] = 0;  // last read after B_{t-1}, next used in round t+2
        }
        if (tid == 0) fcnt[(t + 2) % 3] = 0;              // L_t's length: consumed; refilled in round t+2
        __syncthreads();
        t++;
    }
    if (c == 0 && tid == 0) {
        a.ctl->rounds = t - 1;
        if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
    }
    for (uint32_t i = tid; i < nown; i += CL_THREADS) a.core_mask[v0 + i] = count_of(st[i]) >= k ? 1 : 0;
    cluster.sync();  // no CTA exits while others may still read its shared memory
}

// packed path (k <= 2)
template <int R>
__global__ void __launch_bounds__(PEEL_BLOCK, 4) peel_packed_kernel(PeelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ BlockQueue<uint2> q;
    Ctl *ctl = a.ctl;
    if (ld_cg_u32(&ctl->err) & ERR_BADVERTEX) return;  // uniform across the grid
    if (threadIdx.x == 0) { q.n[0] = 0; q.n[1] = 0; }
    __syncthreads();
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t k = a.k;
    int slot = 0;

    // ---- round 1: F_1 = {v : count(v) < k}, a coalesced scan of the state ----
    // (already emitted by bin_accumulate_kernel when the build was binned)
    if (!a.f1_ready) {
        ull removed = 0;
        scan_emit(a, q, slot, 0, a.n, removed);
        block_add<PEEL_BLOCK>(&ctl->nf[0], removed);
        grid.sync();
    }

    // ---- rounds ----
    uint32_t t = a.t0;
    for (;;) {
        const ull nF = ld_cg_u64(&ctl->nf[(t - 1) % 3]);
        const ull nE = ld_cg_u64(&ctl->ne[(t - 1) % 3]);  // issued before the branch: one round trip
        if (nF == 0) break;
        if (tid == 0) {
            if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
            a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap)] = nF;
            ctl->nf[(t + 1) % 3] = 0;  // round t+2's counters; their last reader finished a barrier ago
            ctl->ne[(t + 1) % 3] = 0;
        }
        const uint2 *Fc = (const uint2 *)a.F[(t - 1) & 1];
        uint2 *Fn = (uint2 *)a.F[t & 1];
        ull *cn = &ctl->ne[t % 3];
        ull kills = 0, crossed = 0;
        if (nE <= nthr) {
            // a latency-bound round (small frontier, e.g. the tail of a near-threshold peel): one
            // entry per thread over the whole grid, and its r-1 decrements issued together before
            // any result is used -- the shortest dependent chain per round
            const uint64_t i = tid;
            const uint2 ent = i < nE ? __ldcg(Fc + i) : make_uint2(0u, 0u);
            bool win = false;
            if (i < nE) {
                const uint32_t bit = 1u << (ent.y & 31);
                win = (atomicAnd(a.alive + (ent.y >> 5), ~bit) & bit) != 0;
            }
            uint32_t ue[R];
            if (win) load_row<R>(a.edges, ent.y, a.m, a.edges_vec, ue);
            const ull dec = 0ull - (((ull)ent.y << 32) + 1ull);
            ull old[R];
            #pragma unroll
            for (int r = 0; r < R; r++) {
                old[r] = ~0ull;  // count 0xFFFFFFFF: never k
                if (win && ue[r] != ent.x) old[r] = atomicAdd(a.state + ue[r], dec);
            }
            kills += win;
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (count_of(old[r]) == k) {
                    crossed++;
                    if (a.peel_round) a.peel_round[ue[r]] = t + 1;
                    bq_push(q, slot, make_uint2(ue[r], idsum_of(old[r]) - ent.y), Fn, cn);
                }
            bq_flush(q, slot, Fn, cn);
            slot ^= 1;
        } else
        for (uint64_t base = (uint64_t)blockIdx.x * CHUNK; base < nE; base += (uint64_t)gridDim.x * CHUNK) {
            // U independent entries per thread, staged so their random accesses overlap
            uint2 ent[U];
            bool win[U];
            #pragma unroll
            for (int j = 0; j < U; j++) {
                const uint64_t i = base + (uint64_t)j * PEEL_BLOCK + threadIdx.x;
                ent[j] = i < nE ? __ldcg(Fc + i) : make_uint2(0u, 0u);
            }
            #pragma unroll
            for (int j = 0; j < U; j++) {  // exactly-once kill of e (P:510-511's concern)
                const uint64_t i = base + (uint64_t)j * PEEL_BLOCK + threadIdx.x;
                win[j] = false;
                if (i < nE) {
                    const uint32_t e = ent[j].y, bit = 1u << (e & 31);
                    win[j] = (atomicAnd(a.alive + (e >> 5), ~bit) & bit) != 0;
                }
            }
            uint32_t ue[U][R];
            #pragma unroll
            for (int j = 0; j < U; j++)
                if (win[j]) {
                    load_row<R>(a.edges, ent[j].y, a.m, a.edges_vec, ue[j]);
                }
            #pragma unroll
            for (int j = 0; j < U; j++)
                if (win[j]) {
                    kills++;
                    const uint32_t e = ent[j].y;
                    const ull dec = 0ull - (((ull)e << 32) + 1ull);
                    #pragma unroll
                    for (int r = 0; r < R; r++) {
                        const uint32_t u = ue[j][r];
                        if (u == ent[j].x) continue;
                        const ull old = atomicAdd(a.state + u, dec);
                        if (count_of(old) == k) {  // count k -> k-1: u joins F_{t+1}
                            crossed++;
                            if (a.peel_round) a.peel_round[u] = t + 1;
                            bq_push(q, slot, make_uint2(u, idsum_of(old) - e), Fn, cn);
                        }
                    }
                }
            bq_flush(q, slot, Fn, cn);
            slot ^= 1;
        }
        block_add<PEEL_BLOCK>(&a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap) + 1], kills);
        block_add<PEEL_BLOCK>(&ctl->nf[t % 3], crossed);
        grid.sync();
        t++;
    }
    if (tid == 0) {
        ctl->rounds = t - 1;
        if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
    }
    write_core_mask<false>(a, tid, nthr);
}

// ---- subround (subtable) variant, P:565-579 -------------------------------------------------
// Vertex classes [c n/r, (c+1) n/r).  Round i = r subrounds; subround j removes the class-j
// vertices whose count is < k at the START of the subround, with their alive edges, after
// subrounds 1..j-1 applied.  Per class c two entry lists (F[b] + c cs, b = 0, 1): the
// "current" list cb[c] gathers class-c crossings until subround c processes it; a class-c
// crossing DURING subround c (possible only when an edge has two class-c vertices) goes to
// the other list, which becomes current afterwards.  cb[] is tracked identically by every
// thread.  Stats are per flattened subround s = (i-1) r + j; the loop stops after a round that
// removes nothing, and `rounds` reports the flattened index of the last non-empty subround.
static constexpr int SUB_QCAP = PEEL_BLOCK;  // one crossing per class per entry in the subtable model
typedef BlockQueueT<uint2, SUB_QCAP, PEEL_BLOCK> SubQ;

template <int R>
__global__ void __launch_bounds__(PEEL_BLOCK) peel_subround_kernel(PeelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ SubQ q[R];
    Ctl *ctl = a.ctl;
    if (ld_cg_u32(&ctl->err) & ERR_BADVERTEX) return;
    #pragma unroll
    for (int c = 0; c < R; c++) bq_init(q[c]);
    __syncthreads();
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t k = a.k;
    const uint64_t cs = a.cs;
    ull *sub = a.sub;  // sub[(c * 2 + b) * 2 + kind]
    uint2 *F0 = (uint2 *)a.F[0], *F1 = (uint2 *)a.F[1];
    auto list = [&](uint32_t c, uint32_t b) { return (b ? F1 : F0) + (uint64_t)c * cs; };
    int slot = 0;
    // initial scan: every vertex with count < k goes to its class's list 0
    {
        ull removed[R];
        #pragma unroll
        for (int c = 0; c < R; c++) removed[c] = 0;
        for (uint64_t base = (uint64_t)blockIdx.x * PEEL_BLOCK; base < a.n; base += (uint64_t)gridDim.x * PEEL_BLOCK) {
            const uint64_t v = base + threadIdx.x;
            const ull w = v < a.n ? ld_cg_u64(a.state + v) : ~0ull;
            const bool in = v < a.n && count_of(w) < k;
            const uint32_t cv = in ? (uint32_t)(v / cs) : 0u;
            #pragma unroll
            for (int c = 0; c < R; c++)
                if (in && cv == (uint32_t)c) {
                    removed[c]++;
                    if (a.peel_round) a.peel_round[v] = (uint32_t)c + 1;  // flattened subround (1, c)
                    if (count_of(w) == 1)
                        bq_push(q[c], slot, make_uint2((uint32_t)v, idsum_of(w)), list(c, 0), &sub[(c * 2 + 0) * 2 + 1]);
                }
            #pragma unroll
            for (int c = 0; c < R; c++) bq_flush(q[c], slot, list(c, 0), &sub[(c * 2 + 0) * 2 + 1]);
            slot ^= 1;
        }
        #pragma unroll
        for (int c = 0; c < R; c++) block_add<PEEL_BLOCK>(&sub[(c * 2 + 0) * 2 + 0], removed[c]);
    }
    grid.sync();
    uint32_t cb[R];
    #pragma unroll
    for (int c = 0; c < R; c++) cb[c] = 0;
    uint32_t flat = 0, last = 0;
    for (;;) {
        bool any = false;
        #pragma unroll 1
        for (uint32_t j = 0; j < (uint32_t)R; j++) {
            flat++;
            const uint32_t cur = cb[j];
            const ull nF = ld_cg_u64(&sub[(j * 2 + cur) * 2 + 0]);
            const ull nE = ld_cg_u64(&sub[(j * 2 + cur) * 2 + 1]);
            if (tid == 0) {
                if (flat <= a.stat_cap) a.rtime[flat - 1] = globaltimer();
                a.stats[2 * (flat <= a.stat_cap ? flat - 1 : a.stat_cap)] = nF;
            }
            ull kills = 0;
            ull xc[R];  // crossings per class this subround
            #pragma unroll
            for (int c = 0; c < R; c++) xc[c] = 0;
            if (nF) {
                any = true;
                last = flat;
                const uint2 *Fc = list(j, cur);
                for (uint64_t base = (uint64_t)blockIdx.x * PEEL_BLOCK; base < nE; base += (uint64_t)gridDim.x * PEEL_BLOCK) {
                    const uint64_t i = base + threadIdx.x;
                    uint32_t cu[R], ce[R], cc[R];
                    bool cv[R];
                    #pragma unroll
                    for (int q2 = 0; q2 < R; q2++) cv[q2] = false;
                    if (i < nE) {
                        const uint2 ent = __ldcg(Fc + i);
                        const uint32_t e = ent.y, bit = 1u << (e & 31);
                        if (atomicAnd(a.alive + (e >> 5), ~bit) & bit) {
                            kills++;
                            const ull dec = 0ull - (((ull)e << 32) + 1ull);
                            uint32_t row[R];
                            load_row<R>(a.edges, e, a.m, a.edges_vec, row);
                            #pragma unroll
                            for (int q2 = 0; q2 < R; q2++) {
                                const uint32_t u = row[q2];
                                if (u == ent.x) continue;
                                const ull old = atomicAdd(a.state + u, dec);
                                if (count_of(old) == k) {
                                    cv[q2] = true;
                                    cu[q2] = u;
                                    ce[q2] = idsum_of(old) - e;
                                    cc[q2] = (uint32_t)(u / cs);
                                }
                            }
                        }
                    }
                    // push crossings, one class at a time (warp-uniform queue selection)
                    #pragma unroll
                    for (int c = 0; c < R; c++) {
                        const uint32_t b = (uint32_t)c == j ? (cb[c] ^ 1u) : cb[c];
                        #pragma unroll
                        for (int q2 = 0; q2 < R; q2++)
                            if (cv[q2] && cc[q2] == (uint32_t)c) {
                                xc[c]++;
                                bq_push(q[c], slot, make_uint2(cu[q2], ce[q2]), list(c, b), &sub[(c * 2 + b) * 2 + 1]);
                            }
                    }
                    #pragma unroll
                    for (int c = 0; c < R; c++) {
                        const uint32_t b = (uint32_t)c == j ? (cb[c] ^ 1u) : cb[c];
                        bq_flush(q[c], slot, list(c, b), &sub[(c * 2 + b) * 2 + 1]);
                    }
                    slot ^= 1;
                }
                if (a.peel_round) {  // removal subround of this list's vertices
                    for (uint64_t i = tid; i < nE; i += nthr) a.peel_round[__ldcg(&Fc[i].x)] = flat;
                }
            }
            block_add<PEEL_BLOCK>(&a.stats[2 * (flat <= a.stat_cap ? flat - 1 : a.stat_cap) + 1], kills);
            #pragma unroll
            for (int c = 0; c < R; c++) {
                const uint32_t b = (uint32_t)c == j ? (cb[c] ^ 1u) : cb[c];
                block_add<PEEL_BLOCK>(&sub[(c * 2 + b) * 2 + 0], xc[c]);
            }
            grid.sync();
            if (tid == 0) {  // this list is consumed; its counters restart (its next append is >= 1 barrier away)
                sub[(j * 2 + cur) * 2 + 0] = 0;
                sub[(j * 2 + cur) * 2 + 1] = 0;
            }
            cb[j] ^= 1u;
        }
        if (!any) break;
    }
    if (tid == 0) {
        ctl->rounds = last;
        if (flat <= a.stat_cap) a.rtime[flat - 1] = globaltimer();
    }
    write_core_mask<false>(a, tid, nthr);
}

// CSR path (any k)
// Peel frontier vertex v (CSR path): kill its alive edges exactly once and decrement their
// other endpoints.  The adjacency list (the static one: dead edges included) is walked in
// chunks of CV entries whose loads, alive tests, kills, row gathers and decrements are each
// issued together, so a chunk costs ~5 dependent memory trips instead of ~2 per entry.
#ifndef PEEL_CV
#define PEEL_CV 4  // C4b rounds: 2/3/4/6/8/16 -> 7.54/7.41/7.36/7.64/7.68/8.94 ms
#endif
static constexpr int CV = PEEL_CV;
template <int R>
__device__ __forceinline__ ull csr_visit(const PeelArgs &a, uint32_t v, uint32_t k, uint32_t t,
                                         BlockQueue<uint32_t> &q, int slot, uint32_t *Fn, ull *cn) {
    ull kills = 0;
    const uint32_t b = v ? __ldg(a.off_end + v - 1) : 0u;
    const uint32_t eend = __ldg(a.off_end + v);
    for (uint32_t p0 = b; p0 < eend; p0 += CV) {
        uint32_t e[CV];
        bool win[CV];
        #pragma unroll
        for (int j = 0; j < CV; j++) e[j] = p0 + j < eend ? __ldg(a.adj + p0 + j) : 0u;
        uint32_t w[CV];
        #pragma unroll
        for (int j = 0; j < CV; j++) w[j] = p0 + j < eend ? ld_cg_u32(a.alive + (e[j] >> 5)) : 0u;
        #pragma unroll
        for (int j = 0; j < CV; j++) {
            const uint32_t bit = 1u << (e[j] & 31);
            win[j] = (w[j] & bit) != 0 && (atomicAnd(a.alive + (e[j] >> 5), ~bit) & bit) != 0;
        }
        uint32_t row[CV][R];
        #pragma unroll
        for (int j = 0; j < CV; j++)
            if (win[j]) load_row<R>(a.edges, e[j], a.m, a.edges_vec, row[j]);
        #pragma unroll
        for (int j = 0; j < CV; j++) {
            if (!win[j]) continue;
            kills++;
            uint32_t old[R];
            #pragma unroll
            for (int r = 0; r < R; r++) old[r] = row[j][r] != v ? atomicSub(a.deg + row[j][r], 1u) : 0u;
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (row[j][r] != v && old[r] == k) {
                    bq_push(q, slot, row[j][r], Fn, cn);
                    if (a.peel_round) a.peel_round[row[j][r]] = t + 1;
                }
        }
    }
    return kills;
}

template <int R>
__global__ void __launch_bounds__(PEEL_BLOCK) peel_csr_kernel(PeelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ BlockQueue<uint32_t> q;
    Ctl *ctl = a.ctl;
    if (ld_cg_u32(&ctl->err) & ERR_BADVERTEX) return;
    if (threadIdx.x == 0) { q.n[0] = 0; q.n[1] = 0; }
    __syncthreads();
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t k = a.k;
    int slot = 0;
    {
        uint32_t *F = (uint32_t *)a.F[0];
        for (uint64_t base = (uint64_t)blockIdx.x * CHUNK; base < a.n; base += (uint64_t)gridDim.x * CHUNK) {
            #pragma unroll
            for (int j = 0; j < U; j++) {
                const uint64_t v = base + (uint64_t)j * PEEL_BLOCK + threadIdx.x;
                if (v < a.n && a.deg[v] < k) {
                    bq_push(q, slot, (uint32_t)v, F, &ctl->ne[0]);
                    if (a.peel_round) a.peel_round[v] = 1;
                }
            }
            bq_flush(q, slot, F, &ctl->ne[0]);
            slot ^= 1;
        }
    }
    grid.sync();
    uint32_t t = 1;
    for (;;) {
        const ull nF = ld_cg_u64(&ctl->ne[(t - 1) % 3]);
        if (nF == 0) break;
        if (tid == 0) {
            if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
            a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap)] = nF;
            ctl->ne[(t + 1) % 3] = 0;
        }
        const uint32_t *Fc = (const uint32_t *)a.F[(t - 1) & 1];
        uint32_t *Fn = (uint32_t *)a.F[t & 1];
        ull *cn = &ctl->ne[t % 3];
        ull kills = 0;
        // one frontier vertex per thread per iteration, grid-stride (C4b rounds: 1/2/4/8 vertices
        // per thread per iteration -> 7.27/7.28/7.37/7.72 ms): no thread walks two adjacency
        // lists in a round that the grid could spread
        for (uint64_t base = (uint64_t)blockIdx.x * PEEL_BLOCK; base < nF; base += (uint64_t)gridDim.x * PEEL_BLOCK) {
            const uint64_t i = base + threadIdx.x;
            if (i < nF) kills += csr_visit<R>(a, ld_cg_u32(Fc + i), k, t, q, slot, Fn, cn);
            bq_flush(q, slot, Fn, cn);
            slot ^= 1;
        }
        block_add<PEEL_BLOCK>(&a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap) + 1], kills);
        grid.sync();
        t++;
    }
    if (tid == 0) {
        ctl->rounds = t - 1;
        if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
    }
    write_core_mask<true>(a, tid, nthr);
}

// frontier-size threshold (fraction of n) above which a round runs binned.  A binned round
// streams the whole 8n-byte state through L2 once; a persistent round pays one random DRAM
// read-modify-write per decrement, whose L2 hit rate falls as 8n outgrows the L2.  Measured
// on B200: n = 10^9 is fastest at 0.02 (0.03..0.006 within noise, 0.05 is
// +6.8 ms), n = 10^8 at 0.05 (0.02 is +0.3 ms).  PEEL_BIN_ROUND_FRAC overrides (0 disables).
static double bin_round_frac(uint64_t n) {
    static double f = -2.0;
    if (f == -2.0) {
        const char *e = getenv("PEEL_BIN_ROUND_FRAC");
        f = e ? atof(e) : -1.0;
    }
    if (f >= 0.0) return f;
    return 8.0 * (double)n >= 2e9 ? 0.02 : 0.05;
}

static unsigned grid_for(uint64_t work, int per_sm = 16) {
    uint64_t blocks = (work + 255) / 256;
    uint64_t cap = (uint64_t)num_sms() * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    return (unsigned)blocks;
}

// cluster size (16, else 8) for peel_cluster_kernel, or 0: the instance's words must fit
// the cluster's shared memory.  PEEL_CLUSTER=0 disables the path (A/B measurement).
static int cluster_eligible(uint64_t n, uint64_t m, const void *kern) {
    const char *ev = getenv("PEEL_CLUSTER");  // read per call: tests toggle it in-process
    if ((ev && atoi(ev) == 0) || n == 0) return 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
    // the launchability answer per (device, kernel, cluster size, shared-memory bytes rounded
    // up to 4 KB) is cached: the occupancy query costs more than a small peel
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int, size_t>, bool> ok;
    static std::map<int, int> optin;
    std::lock_guard<std::mutex> lock(mu);
    if (!optin.count(dev)) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
            cudaGetLastError();
            v = 0;
        }
        optin[dev] = v;
    }
    for (int cs : {CL_MAX, 8}) {
        const ClusterShape shp = cluster_shape(n, m, (uint32_t)cs);
        if (shp.smem + 4096 > (size_t)optin[dev]) continue;  // + static shared memory
        const size_t smem4k = (shp.smem + 4095) & ~(size_t)4095;
        const auto key = std::make_tuple(dev, kern, cs, smem4k);
        // the dynamic-smem attribute: per (device, function), only ever raised (raise_smem)
        if (raise_smem((const void *)kern, smem4k) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        auto it = ok.find(key);
        if (it == ok.end()) {
            bool good = cs <= 8 || cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
            if (good) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)cs);
                cfg.blockDim = dim3(CL_THREADS);
                cfg.dynamicSmemBytes = smem4k;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = (unsigned)cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int nc = 0;
                good = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess && nc >= 1;
            }
            if (!good) cudaGetLastError();
            it = ok.emplace(key, good).first;
        }
        if (it->second) return cs;
    }
    return 0;
}

// read back rounds and per-round statistics after the round loop (one small copy)
static peel_status finish_kcore(uint64_t n, uint32_t cap, uint32_t *rounds, uint64_t *survivors, uint64_t *killed,
                                char *ws, const Layout &L, const PeelArgs &a, cudaStream_t s) {
    ull *stats = (ull *)(ws + L.stats);
    // results: the control block and the first STAT_HEAD rounds' statistics in one copy
    static_assert(sizeof(Ctl) <= 256, "Ctl fits the first 256-byte slot (L.stats follows it)");
    constexpr uint64_t STAT_HEAD = 64;
    std::vector<ull> head((L.stats - L.ctl) / sizeof(ull) + 2 * STAT_HEAD);
    PEEL_CUDA(cudaMemcpyAsync(head.data(), ws + L.ctl, head.size() * sizeof(ull), cudaMemcpyDeviceToHost, s));
    PEEL_CUDA(cudaStreamSynchronize(s));
    prof_collect();
    Ctl hctl;
    memcpy(&hctl, head.data(), sizeof(Ctl));
    if (hctl.err & ERR_BADVERTEX) return PEEL_EINVAL;
    uint64_t T = hctl.rounds;
    if (prof_enabled()) {
        uint64_t nt = (T < STAT_CAP ? T : STAT_CAP - 1) + 1;
        std::vector<ull> rt(nt);
        PEEL_CUDA(cudaMemcpy(rt.data(), a.rtime, sizeof(ull) * nt, cudaMemcpyDeviceToHost));
        std::vector<double> ms(nt > 1 ? nt - 1 : 0);
        for (uint64_t i = 0; i + 1 < nt; i++) ms[i] = (rt[i + 1] - rt[i]) * 1e-6;
        prof_set_rounds(ms);
    }
    *rounds = (uint32_t)T;
    uint64_t nstore = T < cap ? T : cap;
    if (nstore > STAT_CAP) nstore = STAT_CAP;
    if (nstore && (survivors || killed)) {
        const ull *hs = head.data() + (L.stats - L.ctl) / sizeof(ull);
        std::vector<ull> more;
        if (nstore > STAT_HEAD) {
            more.resize(2 * nstore);
            PEEL_CUDA(cudaMemcpy(more.data(), stats, sizeof(ull) * 2 * nstore, cudaMemcpyDeviceToHost));
            hs = more.data();
        }
        uint64_t alive_v = n;
        for (uint64_t t = 0; t < nstore; t++) {
            alive_v -= hs[2 * t];
            if (survivors) survivors[t] = alive_v;
            if (killed) killed[t] = hs[2 * t + 1];
        }
    }
    return (T > cap || T > STAT_CAP) ? PEEL_ETRUNC : PEEL_OK;
}

// peel_kcore_host: the edges arrive from host memory in chunks on a copy stream; the binned
// build partitions each chunk as soon as its copy lands (the partition hides under the
// host->device transfer).  Other paths wait for the whole copy.
struct EdgeStream {
    const uint32_t *host;   // the caller's edges (pinned for the copies to overlap)
    uint32_t *dev;          // = edges of run_kcore
    cudaStream_t copy;
    std::vector<cudaEvent_t> done;  // one per chunk
    uint64_t chunk;         // edges per chunk
};

static peel_status stream_all(const EdgeStream &es, uint64_t m, uint32_t r, cudaStream_t s) {
    for (size_t i = 0; i < es.done.size(); i++) {
        const uint64_t e0 = i * es.chunk, e1 = std::min(m, e0 + es.chunk);
        PEEL_CUDA(cudaMemcpyAsync(es.dev + e0 * r, es.host + e0 * r, sizeof(uint32_t) * r * (e1 - e0),
                                  cudaMemcpyHostToDevice, es.copy));
        PEEL_CUDA(cudaEventRecord(es.done[i], es.copy));
    }
    return PEEL_OK;
}

#include "kcompact.cuh"

// Small instances (the one-cluster path) are launch-bound: the call's memsets, build and round
// loop are captured once per (device, stream, buffers, shape) into a CUDA graph and replayed
// (PEEL_GRAPH=0 disables).  A few entries are kept; a new shape or buffer evicts the oldest.
struct SmallGraph {
    int dev;
    const void *edges, *mask, *pr, *ws;
    cudaStream_t s;
    uint64_t n, m;
    uint32_t r, k;
    cudaGraphExec_t exec;
};

static bool graphs_on() {
    const char *e = getenv("PEEL_GRAPH");
    return !(e && atoi(e) == 0);
}

template <int R>
static peel_status run_kcore(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t k, bool csr, uint32_t flags,
                             uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors,
                             uint64_t *killed, uint32_t cap, uint32_t *peel_round, char *ws,
                             const Layout &L, cudaStream_t s, const EdgeStream *es = nullptr,
                             bool capturing = false);

template <int R>
static peel_status run_small_graph(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t k, uint8_t *core_mask,
                                   uint32_t *rounds, uint64_t *survivors, uint64_t *killed, uint32_t cap,
                                   uint32_t *peel_round, char *ws, const Layout &L, cudaStream_t s) {
    static std::mutex mu;
    static std::vector<SmallGraph> cache;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    PEEL_CUDA(cudaGetDevice(&dev));
    cudaGraphExec_t exec = nullptr;
    for (auto &g : cache)
        if (g.dev == dev && g.edges == edges && g.mask == core_mask && g.pr == peel_round && g.ws == ws && g.s == s &&
            g.n == n && g.m == m && g.r == (uint32_t)R && g.k == k) {
            exec = g.exec;
            break;
        }
    if (!exec) {
        // captured on a private stream (the caller's may be the legacy default stream, which
        // cannot be captured); the graph is then launched into the caller's stream
        static std::map<int, cudaStream_t> cap_stream;
        if (!cap_stream.count(dev)) {
            cudaStream_t cs = nullptr;
            PEEL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cap_stream[dev] = cs;
        }
        cudaStream_t cs = cap_stream[dev];
        cudaGraph_t graph = nullptr;
        PEEL_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        prof_capture(true);
        peel_status st = run_kcore<R>(edges, n, m, k, false, 0u, core_mask, rounds, survivors, killed, cap, peel_round,
                                      ws, L, cs, nullptr, true);
        prof_capture(false);
        const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        if (st != PEEL_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (ce != cudaSuccess) { set_cuda_error(ce, "cudaStreamEndCapture"); return PEEL_ECUDA; }
        const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) { set_cuda_error(ie, "cudaGraphInstantiate"); return PEEL_ECUDA; }
        if (cache.size() >= 8) {
            cudaGraphExecDestroy(cache.front().exec);
            cache.erase(cache.begin());
        }
        cache.push_back({dev, edges, core_mask, peel_round, ws, s, n, m, (uint32_t)R, k, exec});
    }
    {
        ProfScope ps("peel_small_graph", s);
        PEEL_CUDA(cudaGraphLaunch(exec, s));
    }
    prof_add_launches(m ? 1 : 0);  // build + round loop inside the graph (ProfScope counted one)
    PeelArgs a;
    memset(&a, 0, sizeof a);
    a.rtime = (ull *)(ws + L.rtime);
    return finish_kcore(n, cap, rounds, survivors, killed, ws, L, a, s);
}

template <int R>
static peel_status run_kcore(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t k, bool csr, uint32_t flags,
                             uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors,
                             uint64_t *killed, uint32_t cap, uint32_t *peel_round, char *ws,
                             const Layout &L, cudaStream_t s, const EdgeStream *es, bool capturing) {
    const bool subr = (flags & PEEL_FLAG_SUBROUNDS) != 0;
    if (!capturing && !csr && !subr && !es && !L.nbins && graphs_on() &&
        cluster_eligible(n, m, (const void *)peel_cluster_kernel<R>))
        return run_small_graph<R>(edges, n, m, k, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s);
    Ctl *ctl = (Ctl *)(ws + L.ctl);
    ull *stats = (ull *)(ws + L.stats);
    uint32_t *alive = (uint32_t *)(ws + L.alive);
    PEEL_CUDA(cudaMemsetAsync(ws + L.ctl, 0, L.state ? L.state - L.ctl : L.deg - L.ctl, s));
    PEEL_CUDA(cudaMemsetAsync(alive, 0xFF, sizeof(uint32_t) * ((m + 31) / 32), s));

    PeelArgs a;
    memset(&a, 0, sizeof a);
    a.edges = edges; a.n = n; a.m = m; a.k = k;
    a.stat_cap = STAT_CAP;
    a.alive = alive;
    a.F[0] = ws + L.F0;
    a.F[1] = ws + L.F1;
    a.ctl = ctl; a.stats = stats;
    a.rtime = (ull *)(ws + L.rtime);
    a.core_mask = core_mask; a.peel_round = peel_round;
    a.mask_vec = ((uintptr_t)core_mask & 15) == 0;
    a.edges_vec = ((uintptr_t)edges & 15) == 0;
    if (peel_round) PEEL_CUDA(cudaMemsetAsync(peel_round, 0, sizeof(uint32_t) * n, s));

    if (es) {
        peel_status st = stream_all(*es, m, R, s);
        if (st != PEEL_OK) return st;
        if (csr || !L.nbins)  // only the binned build consumes the chunks as they land
            for (auto ev : es->done) PEEL_CUDA(cudaStreamWaitEvent(s, ev, 0));
    }
    bool compact_done = false;
    if (!csr && !subr && L.compact && compact_on()) {
        bool fallback = false;
        peel_status st = run_compact<R>(edges, n, m, k, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s,
                                        es, a, &fallback);
        if (!fallback) return st;
        // a bin overflowed: the uncompacted binned path below rebuilds from scratch
        PEEL_CUDA(cudaMemsetAsync(ws + L.ctl, 0, L.state - L.ctl, s));
        es = nullptr;  // the copies have landed (the partition waited for every chunk)
        compact_done = false;
    }
    (void)compact_done;
    if (!csr && L.nbins) {
        // binned build: partition endpoint increments by vertex bin, accumulate each bin in L2
        ull *state = (ull *)(ws + L.state);
        a.state = state;
        ull *cursor = (ull *)(ws + L.bin_cursor), *bbase = (ull *)(ws + L.bin_base), *bcap = (ull *)(ws + L.bin_cap);
        ull *entries = (ull *)(ws + L.entries);
        {
            ProfScope ps("bin_init", s);
            bin_init_kernel<<<1, 32, 0, s>>>(n, n, m, R, L.nbins, cursor, bbase, bcap);
        }
        const size_t smem = partition_smem(R, L.nbins);
        PEEL_CUDA(raise_smem((const void *)bin_partition_kernel<R>, smem));
        int pblocks = 0;
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pblocks, bin_partition_kernel<R>, PART_BLOCK, smem));
        if (pblocks < 1) pblocks = 1;
        if (m && !es) {
            ProfScope ps("bin_partition", s);
            bin_partition_kernel<R><<<num_sms() * pblocks, PART_BLOCK, smem, s>>>(edges, n, m, (uint32_t)L.nbins, cursor, bbase,
                                                                                   bcap, entries, &ctl->err, &ctl->binovf,
                                                                                   0ull, n, 0ull);
        } else if (m) {  // chunk by chunk, each after its copy
            for (size_t i = 0; i < es->done.size(); i++) {
                const uint64_t e0 = i * es->chunk, e1 = std::min(m, e0 + es->chunk);
                PEEL_CUDA(cudaStreamWaitEvent(s, es->done[i], 0));
                ProfScope ps("bin_partition", s);
                bin_partition_kernel<R><<<num_sms() * pblocks, PART_BLOCK, smem, s>>>(edges, n, e1, (uint32_t)L.nbins, cursor,
                                                                                       bbase, bcap, entries, &ctl->err,
                                                                                       &ctl->binovf, 0ull, n, e0);
            }
        }
        PEEL_CUDA(cudaGetLastError());
        BinArgs bn;
        bn.nbins = L.nbins; bn.cursor = cursor; bn.base = bbase; bn.cap = bcap; bn.entries = entries;
        int per_sm = 0;
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bin_accumulate_kernel<R>, PEEL_BLOCK, 0));
        if (per_sm < 1) per_sm = 1;
        void *bargs[] = {&a, &bn};
        {
            ProfScope ps("bin_accumulate", s);
            PEEL_CUDA(cudaLaunchCooperativeKernel((void *)bin_accumulate_kernel<R>, num_sms() * per_sm, PEEL_BLOCK,
                                                  bargs, 0, s));
        }
        a.f1_ready = 1;
    } else if (!csr) {
        ull *state = (ull *)(ws + L.state);
        PEEL_CUDA(cudaMemsetAsync(state, 0, sizeof(ull) * n, s));
        a.state = state;
        if (m) {
            ProfScope ps("build_packed", s);
            build_packed_kernel<R><<<grid_for(m), 256, 0, s>>>(edges, n, m, state, ctl);
        }
    } else {
        uint32_t *deg = (uint32_t *)(ws + L.deg);
        uint32_t *off = (uint32_t *)(ws + L.off);
        uint32_t *bsum = (uint32_t *)(ws + L.bsum);
        uint32_t *adj = (uint32_t *)(ws + L.adj);
        PEEL_CUDA(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * n, s));
        const bool binned = L.nbins > 0 && m > 0;
        bool scatter_from_bins = false;
        ull *cursor = (ull *)(ws + L.bin_cursor), *bbase = (ull *)(ws + L.bin_base), *bcap = (ull *)(ws + L.bin_cap);
        ull *entries = (ull *)(ws + L.entries);
        uint64_t maxcap = 0;
        for (uint64_t b = 0; b < L.nbins; b++) maxcap = std::max<uint64_t>(maxcap, bin_capacity(n, n, m, R, b));
        const dim3 bgrid((unsigned)((maxcap + 256 * CSRB_PER - 1) / (256 * CSRB_PER)), (unsigned)L.nbins);
        if (binned) {
            {
                ProfScope ps("bin_init", s);
                bin_init_kernel<<<1, 32, 0, s>>>(n, n, m, R, L.nbins, cursor, bbase, bcap);
            }
            const size_t smem = partition_smem(R, L.nbins);
            PEEL_CUDA(raise_smem((const void *)bin_partition_kernel<R>, smem));
            int pblocks = 0;
            PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pblocks, bin_partition_kernel<R>, PART_BLOCK, smem));
            pblocks = pblocks < 1 ? 1 : pblocks;
            {
                ProfScope ps("bin_partition", s);
                bin_partition_kernel<R><<<num_sms() * pblocks, PART_BLOCK, smem, s>>>(edges, n, m, (uint32_t)L.nbins,
                                                                                       cursor, bbase, bcap, entries, &ctl->err,
                                                                                       &ctl->binovf, 0ull, n, 0ull);
            }
            // a bin overflow (adversarial degree skew) only loses entries of the binned copy:
            // fall back to the direct histogram below if it happened (checked on the host)
            Ctl h;
            PEEL_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
            PEEL_CUDA(cudaStreamSynchronize(s));
            if (h.err) return PEEL_EINVAL;
            if (!h.binovf) {
                ProfScope ps("csr_bin_deg", s);
                csr_bin_deg_kernel<<<bgrid, 256, 0, s>>>(entries, bbase, cursor, deg);
            }
            if (h.binovf) {
                ProfScope ps("build_deg", s);
                build_deg_kernel<R><<<grid_for(m), 256, 0, s>>>(edges, n, m, deg, ctl);
            }
            scatter_from_bins = !h.binovf;
        } else if (m) {
            ProfScope ps("build_deg", s);
            build_deg_kernel<R><<<grid_for(m), 256, 0, s>>>(edges, n, m, deg, ctl);
        }
        uint64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
        {
            ProfScope ps("scan_tiles", s);
            scan_tiles_kernel<<<(unsigned)nb, PEEL_BLOCK, 0, s>>>(deg, n, off, bsum);
        }
        {
            ProfScope ps("scan_bsum", s);
            scan_bsum_kernel<<<1, PEEL_BLOCK, 0, s>>>(bsum, nb);
        }
        {
            ProfScope ps("scan_add", s);
            scan_add_kernel<<<grid_for(n), PEEL_BLOCK, 0, s>>>(off, n, bsum);
        }
        if (scatter_from_bins) {
            ProfScope ps("csr_bin_scatter", s);
            csr_bin_scatter_kernel<<<dim3(bgrid.x, bgrid.y << CSR_SUB_LOG), 256, 0, s>>>(entries, bbase, cursor, off, adj);
        } else if (m) {
            ProfScope ps("scatter", s);
            scatter_kernel<R><<<grid_for(m), 256, 0, s>>>(edges, n, m, off, adj);
        }
        a.deg = deg; a.off_end = off; a.adj = adj;
    }
    PEEL_CUDA(cudaGetLastError());

    // binned rounds while the frontier is a large fraction of n (see round_apply_kernel)
    a.t0 = 1;
    if (!csr && !subr && L.nbins && bin_round_frac(n) > 0.0) {
        ull *cursor = (ull *)(ws + L.bin_cursor);
        BinRound br;
        br.nbins = (uint32_t)L.nbins;
        br.cursor = cursor;
        br.base = (const ull *)(ws + L.bin_base);
        br.entries = (ull *)(ws + L.entries);
        br.work = &ctl->work;
        const size_t ksmem = kill_partition_smem(R, br.nbins);
        PEEL_CUDA(raise_smem((const void *)round_kill_partition_kernel<R>, ksmem));
        // keep >= 60 KB of L1 for the row gathers: with the shared-memory carve-out at 86-100%
        // (28 KB L1 or less) the C5 kill phase takes 43 ms instead of 24.5 (72% and 58%: 24.5-24.7)
        PEEL_CUDA(cudaFuncSetAttribute(round_kill_partition_kernel<R>, cudaFuncAttributePreferredSharedMemoryCarveout, 72));
        int kb = 0, db = 0;
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&kb, round_kill_partition_kernel<R>, PART_BLOCK, ksmem));
        // frontier sort by edge bin before each kill phase (PEEL_ESORT=0 disables, for A/B)
        const char *esv = getenv("PEEL_ESORT");
        const bool esort = !(esv && atoi(esv) == 0) && m > 0;
        const uint32_t enb = (uint32_t)((m + (1ull << EB_SHIFT) - 1) >> EB_SHIFT);
        // D also histograms F_{t+1} by edge bin, so rounds after the first skip the hist pass
        const size_t dsmem = sizeof(uint32_t) * (br.nbins + 1) + (esort ? sizeof(uint32_t) * enb : 0);
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&db, round_apply_kernel, PEEL_BLOCK, dsmem));
        kb = kb < 1 ? 1 : kb;
        db = db < 1 ? 1 : db;
        br.ehist = nullptr;
        br.enb = enb;
        // F_t's edge-bin histogram lives in ehist[t & 1]; round t's D fills ehist[(t + 1) & 1]
        ull *ehist[2] = {(ull *)(ws + L.esort), (ull *)(ws + L.esort) + enb + 1};
        ull *ecur = ehist[1] + enb + 1;
        const size_t essmem = esort_scatter_smem(enb);
        if (esort) {
            PEEL_CUDA(cudaMemsetAsync(ehist[1], 0, sizeof(ull) * (enb + 1), s));
            PEEL_CUDA(raise_smem((const void *)esort_scatter_kernel, essmem));
        }
        br.Fsrc = nullptr;
        uint32_t t = 1;
        for (;;) {
            Ctl h;
            PEEL_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
            PEEL_CUDA(cudaStreamSynchronize(s));
            if (h.err) break;  // the persistent kernel reports it
            // an overflowed build bin bounds nothing: a round's decrements of bin b are a
            // subset of the build's entries of bin b, which did not fit its capacity
            if (h.binovf) break;
            const ull nF = h.nf[(t - 1) % 3], nE = h.ne[(t - 1) % 3];
            if (nF == 0 || (double)nE < bin_round_frac(n) * (double)n) break;
            PEEL_CUDA(cudaMemsetAsync(cursor, 0, sizeof(ull) * L.nbins, s));
            PEEL_CUDA(cudaMemsetAsync(&ctl->work, 0, sizeof(ull), s));
            br.t = t;
            br.Fsrc = nullptr;
            if (esort) {
                const uint2 *src = (const uint2 *)a.F[(t - 1) & 1];
                uint2 *dst = (uint2 *)a.F[t & 1];  // free until this round's apply writes F_{t+1}
                const ull *pN = &ctl->ne[(t - 1) % 3];
                ProfScope ps("frontier_edge_sort", s);
                if (!br.ehist)  // round 1: F_1 came from the build; later rounds' D made the histogram
                    esort_hist_kernel<<<grid_for(nE, 8), 256, sizeof(uint32_t) * enb, s>>>(src, pN, enb, ehist[t & 1]);
                PEEL_CUDA(cudaMemsetAsync(ecur, 0, sizeof(ull) * enb, s));
                PEEL_CUDA(cudaMemsetAsync(ehist[(t + 1) & 1], 0, sizeof(ull) * enb, s));  // for this round's D
                const uint64_t chunks = (nE + ES_CH - 1) / ES_CH;
                const unsigned sg = (unsigned)std::min<uint64_t>(chunks, (uint64_t)num_sms() * ES_BLOCKS);
                esort_scatter_kernel<<<sg ? sg : 1, 256, essmem, s>>>(src, pN, enb, ehist[t & 1], ecur, dst);
                br.Fsrc = dst;
                br.ehist = ehist[(t + 1) & 1];
            }
            {
                ProfScope ps("round_kill_partition", s);
                round_kill_partition_kernel<R><<<num_sms() * kb, PART_BLOCK, ksmem, s>>>(a, br);
            }
            {
                ProfScope ps("round_apply", s);
                round_apply_kernel<<<num_sms() * db, PEEL_BLOCK, dsmem, s>>>(a, br);
            }
            PEEL_CUDA(cudaGetLastError());
            t++;
        }
        a.t0 = t;
    }

    // small packed instances: the whole round loop in one cluster's shared memory
    if (!csr && !subr && a.t0 == 1 && !L.nbins) {
        const int cl = cluster_eligible(n, m, (const void *)peel_cluster_kernel<R>);
        if (cl) {
            const ClusterShape shp = cluster_shape(n, m, (uint32_t)cl);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)cl);
            cfg.blockDim = dim3(CL_THREADS);
            cfg.dynamicSmemBytes = shp.smem;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            {
                ProfScope ps("peel_rounds_cluster", s);
                PEEL_CUDA(cudaLaunchKernelEx(&cfg, peel_cluster_kernel<R>, a, shp));
            }
            if (capturing) return PEEL_OK;  // run_small_graph launches the graph, then finishes
            return finish_kcore(n, cap, rounds, survivors, killed, ws, L, a, s);
        }
    }

    // cooperative persistent round loop: every block must be co-resident
    void *kern = csr ? (void *)peel_csr_kernel<R> : (subr ? (void *)peel_subround_kernel<R> : (void *)peel_packed_kernel<R>);
    if (subr) {
        a.r = R;
        a.cs = n / R;
        a.sub = (ull *)(ws + L.sub);
    }
    int per_sm = 0;
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PEEL_BLOCK, 0));
    if (per_sm < 1) per_sm = 1;
    unsigned grid = (unsigned)(num_sms() * per_sm);
    // small instances: no more blocks than one CHUNK of vertices each (cheaper grid barriers)
    const uint64_t want = (n + CHUNK - 1) / CHUNK;
    if (want < grid) grid = (unsigned)(want < (uint64_t)num_sms() ? num_sms() : want);
    void *args[] = {&a};
    {
        ProfScope ps(csr ? "peel_rounds_csr" : (subr ? "peel_subrounds" : "peel_rounds_packed"), s);
        PEEL_CUDA(cudaLaunchCooperativeKernel(kern, grid, PEEL_BLOCK, args, 0, s));
    }

    return finish_kcore(n, cap, rounds, survivors, killed, ws, L, a, s);
}

static bool kcore_args_ok(uint64_t n, uint64_t m, uint32_t r, bool csr) {
    if (r < 2 || r > 8 || n > (1ull << 32) || m >= (1ull << 32)) return false;
    if (csr && (uint64_t)r * m >= (1ull << 32)) return false;
    return true;
}

static bool use_csr(uint32_t k, uint32_t flags) { return (flags & PEEL_FLAG_CSR) || k >= 3; }

// ---- the binned build for one vertex shard (shard.h; used by dist.cu) --------------------
struct ShardBins {
    uint64_t nbins, total_cap;
    size_t cursor, base, cap, flag, ctl, esort, entries, total;
};

static ShardBins shard_bins(uint64_t n, uint64_t m, uint32_t r, uint64_t nloc) {
    ShardBins B;
    B.nbins = (nloc + (1ull << BIN_SHIFT) - 1) >> BIN_SHIFT;
    B.total_cap = 0;
    for (uint64_t b = 0; b < B.nbins; b++) B.total_cap += bin_capacity(n, nloc, m, r, b);
    size_t o = 0;
    B.cursor = o; o += al(sizeof(ull) * B.nbins);
    B.base = o; o += al(sizeof(ull) * B.nbins);
    B.cap = o; o += al(sizeof(ull) * B.nbins);
    B.flag = o; o += al(sizeof(uint32_t) + 8 + sizeof(ull));  // overflow flag, then the D work counter
    B.ctl = o; o += al(sizeof(Ctl));                           // binned rounds: round_apply's counters
    B.esort = o; o += al(sizeof(ull) * 2 * (((m + (1ull << EB_SHIFT) - 1) >> EB_SHIFT) + 1));  // edge sort
    B.entries = o; o += al(sizeof(ull) * B.total_cap);
    B.total = o;
    return B;
}

size_t shard_build_bytes(uint64_t n, uint64_t m, uint32_t r, uint64_t nloc) {
    if (nloc <= BIN_MIN_N || r < 2 || r > 8) return 0;
    return shard_bins(n, m, r, nloc).total;
}

// ---- narrow shards (v1 - v0 <= n / 4; dist.cu at P >= 4): the replicated edge list is read
// by every shard, and bin_partition_kernel's per-chunk work (staging, validation, ranking, one
// scan and one global atomic per bin, the write-out) is paid per 1024 edges however few of
// their endpoints the shard keeps (C5 over 8 virtual shards: 6.4 ms per shard against 10 ms
// for all endpoints).  Instead: (1) a streaming filter pass -- each block walks a fixed edge
// range, validates every edge and appends the shard's endpoints (e << 32 | local id) to its own
// region of a scratch buffer (warp ballots, one shared-memory counter; no global atomics);
// (2) the regions' entries are counting-sorted into the shard's bins chunk by chunk, as
// bin_partition_kernel sorts its chunks.  A region that overflows (adversarial skew) sends the
// build back to bin_partition_kernel.
static constexpr int SF_U = 4;          // edges per thread per step
static constexpr int SB_CH = 2048;      // entries per binning chunk
struct SFHead {                         // at the start of the scratch buffer
    uint32_t ovf;
    uint32_t pad[63];
};

#ifndef PEEL_SF_MINB
#define PEEL_SF_MINB 6
#endif
template <int R>
__global__ void __launch_bounds__(256, PEEL_SF_MINB) shard_filter_kernel(const uint32_t *__restrict__ edges, uint64_t n, uint64_t m,
                                                           uint64_t v0, uint64_t v1, uint64_t per_block, ull *out,
                                                           uint64_t cap_b, ull *counts, uint32_t *err, uint32_t *ovf,
                                                           int vec) {
    // a warp takes 128 edges (R * 32 16-byte words) per step: coalesced 16-byte loads staged in
    // its own shared-memory slice, then lane l validates and filters edges 4 l .. 4 l + 3
    // (scalar loads with a 12-byte lane stride cost three times the L1 wavefronts: 5.2 ms per
    // C5 shard against the 1.4 ms the bytes take)
    constexpr int WW = 32 * R;  // 16-byte words per warp step (128 edges)
    __shared__ __align__(16) uint32_t stage[8][2][4 * WW];  // per warp, double-buffered
    __shared__ uint32_t cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const uint64_t e_lo = (uint64_t)blockIdx.x * per_block, e_hi = min(m, e_lo + per_block);
    ull *ob = out + (uint64_t)blockIdx.x * cap_b;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t wend = m * R;  // words in the array
    const uint32_t nm1 = (uint32_t)(n - 1), lv0 = (uint32_t)v0, nl32 = (uint32_t)(v1 - v0);
    bool over = false, bad = false;
    // the step's R 16-byte words per lane into stage[w][buf]: cp.async (no registers held, the
    // next step's copy in flight while this one is filtered); scalar loads at the array's end
    auto fetch = [&](uint64_t base, int buf) {
        const uint64_t w0 = base * R;  // a multiple of 4 R words: 16-byte aligned
        #pragma unroll
        for (int q = 0; q < R; q++) {
            const uint64_t wi = w0 + 4 * (uint64_t)(q * 32 + lane);
            uint32_t *dst = &stage[w][buf][4 * (q * 32 + lane)];
            if (vec && wi + 4 <= wend) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(edges + wi) : "memory");
            } else {
                #pragma unroll
                for (int x = 0; x < 4; x++) dst[x] = wi + x < wend ? __ldcs(edges + wi + x) : 0u;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const uint64_t step = 8 * 128;
    uint64_t base = e_lo + (uint64_t)w * 128;
    if (base < e_hi) fetch(base, 0);
    for (int buf = 0; base < e_hi; base += step, buf ^= 1) {
        if (base + step < e_hi) fetch(base + step, buf ^ 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");  // keep one group per step
        asm volatile("cp.async.wait_group 1;" ::: "memory");       // this step's copies landed
        __syncwarp();
        const uint32_t *sw = stage[w][buf];
        uint32_t wd[4 * R];
        #pragma unroll
        for (int q = 0; q < R; q++) {
            const uint4 v = reinterpret_cast<const uint4 *>(sw)[lane * R + q];
            wd[4 * q] = v.x; wd[4 * q + 1] = v.y; wd[4 * q + 2] = v.z; wd[4 * q + 3] = v.w;
        }
        __syncwarp();  // every lane read buf before the step after next refills it
        // each lane's kept words (32-bit compares: n <= 2^32, nloc < 2^32), a warp scan of the
        // per-lane counts, ONE shared-memory reservation per warp step; a lane writes its kept
        // words contiguously (the order inside a region is free: the binning pass sorts)
        uint32_t keep = 0;  // bit R j + q: word q of the lane's edge j is the shard's
        const uint32_t nin = (uint32_t)min((uint64_t)128, e_hi - base);  // edges of the step
        #pragma unroll
        for (int j = 0; j < 4; j++) {
            const bool inb = 4 * lane + j < nin;
            bool valid = true;
            #pragma unroll
            for (int q = 0; q < R; q++) valid &= wd[R * j + q] <= nm1;
            #pragma unroll
            for (int q = 0; q < R; q++)
                #pragma unroll
                for (int q2 = q + 1; q2 < R; q2++) valid &= wd[R * j + q] != wd[R * j + q2];
            bad |= inb && !valid;
            uint32_t kj = 0;
            #pragma unroll
            for (int q = 0; q < R; q++) kj |= (uint32_t)(wd[R * j + q] - lv0 < nl32) << q;
            keep |= (inb && valid ? kj : 0u) << (R * j);
        }
        const uint32_t c = __popc(keep);
        uint32_t incl = c;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot) {  // warp-uniform
            uint32_t run = 0;
            if (lane == 0) run = atomicAdd(&cnt, tot);
            run = __shfl_sync(0xffffffffu, run, 0) + incl - c;
            const ull eb = (ull)(base + 4 * lane) << 32;
            for (uint32_t kk = keep; kk; kk &= kk - 1, run++) {  // the lane's kept words, in order
                const uint32_t x = __ffs(kk) - 1, j = x / R;
                uint32_t u = 0;  // wd[x] with constant register indices (a dynamic index spills wd)
                #pragma unroll
                for (int y = 0; y < 4 * R; y++) u = x == (uint32_t)y ? wd[y] : u;
                if (run < cap_b) ob[run] = (eb + ((ull)j << 32)) | (u - lv0);
                else over = true;
            }
        }
    }
    if (bad) atomicOr(err, ERR_BADVERTEX);
    if (over) atomicOr(ovf, 1u);
    __syncthreads();
    if (threadIdx.x == 0) counts[blockIdx.x] = min((uint64_t)cnt, cap_b);
}

// chunk c of the regions' entries: region c / cpr, entries [(c % cpr) SB_CH, +SB_CH)
__global__ void __launch_bounds__(256, 5) shard_bin_kernel(const ull *__restrict__ in, uint64_t cap_b,
                                                           const ull *__restrict__ counts, uint64_t nchunks,
                                                           uint64_t cpr, uint32_t nbins, ull *cursor,
                                                           const ull *__restrict__ base, const ull *__restrict__ cap,
                                                           ull *entries, uint32_t *binovf) {
    extern __shared__ unsigned char smem_raw[];
    ull *sent = (ull *)smem_raw;                  // [SB_CH]
    ull *gpos = sent + SB_CH;                     // [nbins]
    uint32_t *hist = (uint32_t *)(gpos + nbins);  // [nbins]
    uint32_t *offs = hist + nbins;
    uint32_t *fill = offs + nbins;
    __shared__ uint32_t total;
    constexpr int PER = SB_CH / 256;
    const ull mask = (1ull << BIN_SHIFT) - 1;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const uint64_t reg = c / cpr, off = (c % cpr) * SB_CH;
        const uint64_t cntr = counts[reg];
        if (off >= cntr) continue;  // uniform
        const uint32_t ne = (uint32_t)min((uint64_t)SB_CH, cntr - off);
        const ull *src = in + reg * cap_b + off;
        for (uint32_t b = threadIdx.x; b < nbins; b += 256) hist[b] = 0;
        __syncthreads();
        ull x[PER];
        uint32_t rk[PER];
        #pragma unroll
        for (int q = 0; q < PER; q++) {
            const uint32_t i = q * 256 + threadIdx.x;
            x[q] = i < ne ? __ldcs(src + i) : 0ull;
        }
        #pragma unroll
        for (int q = 0; q < PER; q++)
            if (q * 256 + threadIdx.x < ne) rk[q] = atomicAdd(&hist[(uint32_t)x[q] >> BIN_SHIFT], 1u);
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t per = (nbins + 31) / 32;
            uint32_t loc = 0;
            for (uint32_t q = 0; q < per; q++) {
                const uint32_t b = threadIdx.x * per + q;
                loc += b < nbins ? hist[b] : 0;
            }
            uint32_t y = loc;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
                if ((int)threadIdx.x >= o) y += z;
            }
            uint32_t run = y - loc;
            for (uint32_t q = 0; q < per; q++) {
                const uint32_t b = threadIdx.x * per + q;
                if (b < nbins) { offs[b] = run; run += hist[b]; }
            }
            if (threadIdx.x == 31) total = y;
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nbins; b += 256)
            if (hist[b]) {
                const ull g = atomicAdd(cursor + b, (ull)hist[b]);
                const ull cp = cap[b];
                if (g + hist[b] > cp) atomicOr(binovf, 1u);
                gpos[b] = base[b] + g;
                fill[b] = (uint32_t)(g >= cp ? 0ull : min((ull)hist[b], cp - g));
            }
        #pragma unroll
        for (int q = 0; q < PER; q++)
            if (q * 256 + threadIdx.x < ne) sent[offs[(uint32_t)x[q] >> BIN_SHIFT] + rk[q]] = x[q];
        __syncthreads();
        const uint32_t tot = total;
        for (uint32_t i = threadIdx.x; i < tot; i += 256) {
            const ull v = sent[i];
            const uint32_t b = (uint32_t)v >> BIN_SHIFT;
            const uint32_t q = i - offs[b];
            if (q < fill[b]) entries[gpos[b] + q] = v & ~(0xFFFFFFFFull ^ mask);
        }
        __syncthreads();
    }
}

static size_t shard_bin_smem(uint64_t nbins) { return sizeof(ull) * SB_CH + (sizeof(ull) + 3 * sizeof(uint32_t)) * nbins; }

// the filter path's geometry: blocks, edges per block, region capacity (expected endpoints of
// the shard in a block's edges + 8 standard deviations + 4096), bytes of scratch it needs
struct SFGeom {
    uint64_t nblk, per_block, cap_b, cpr;
    size_t bytes;
};
static SFGeom sf_geom(uint64_t n, uint64_t m, uint32_t r, uint64_t nloc, int per_sm) {
    SFGeom g;
    g.nblk = (uint64_t)num_sms() * (per_sm < 1 ? 1 : per_sm);  // one resident wave
    g.per_block = (((m + g.nblk - 1) / g.nblk) + 127) & ~127ull;  // whole 128-edge warp steps
    const double lam = (double)g.per_block * r * (double)nloc / (double)n;
    g.cap_b = (uint64_t)(lam + 8.0 * sqrt(lam)) + 4096;
    const char *ce = getenv("PEEL_SHARD_FILTER_CAP");  // tests: a small region forces the fallback
    if (ce && atoll(ce) > 0) g.cap_b = (uint64_t)atoll(ce);
    g.cpr = (g.cap_b + SB_CH - 1) / SB_CH;
    g.bytes = sizeof(SFHead) + al(sizeof(ull) * g.nblk) + sizeof(ull) * g.nblk * g.cap_b;
    return g;
}

// the shard's accumulation and F_1 in one cooperative pass (round 2), as cbuild_kernel does for
// one GPU: per bin, zero its states in L2, grid barrier, the bin's entries as REDs (8 loads in
// flight per thread), grid barrier, then scan it -- still in L2 -- for F_1 (count < k; entries
// (v0 + i, id sum) for count 1) while the next bin is zeroed.  Replaces the 8 nloc-byte memset,
// bin_red_kernel and dist.cu's scan, which re-read the state from DRAM.
static constexpr int SA_SU = 4;  // states per thread per scan step
__global__ void __launch_bounds__(256) shard_accum_kernel(const ull *__restrict__ entries, const ull *__restrict__ base,
                                                          const ull *__restrict__ cursor, uint32_t nbins, uint64_t nloc,
                                                          uint64_t v0, uint32_t k, ull *state, uint2 *F, ull *ne,
                                                          ull *nf) {
    cg::grid_group grid = cg::this_grid();
    typedef BlockQueueT<uint2, 4 * 256, 256> Q;
    __shared__ Q q;
    bq_init(q);
    __syncthreads();
    const uint64_t tid = blockIdx.x * 256ull + threadIdx.x, nthr = (uint64_t)gridDim.x * 256;
    const ull mask = (1ull << BIN_SHIFT) - 1;
    ull removed = 0;
    int slot = 0;
    for (uint32_t b = 0; b <= nbins; b++) {
        if (b > 0) {  // scan bin b - 1 (in L2)
            const uint64_t lo = (uint64_t)(b - 1) << BIN_SHIFT, hi = min(nloc, lo + ((uint64_t)1 << BIN_SHIFT));
            for (uint64_t s0 = lo + (uint64_t)blockIdx.x * 256 * SA_SU; s0 < hi; s0 += (uint64_t)gridDim.x * 256 * SA_SU) {
                ull w[SA_SU];
                #pragma unroll
                for (int j = 0; j < SA_SU; j++) {
                    const uint64_t i = s0 + (uint64_t)j * 256 + threadIdx.x;
                    w[j] = i < hi ? __ldcg(state + i) : ~0ull;
                }
                #pragma unroll
                for (int j = 0; j < SA_SU; j++) {
                    const uint64_t i = s0 + (uint64_t)j * 256 + threadIdx.x;
                    if ((uint32_t)w[j] < k) {
                        removed++;
                        if ((uint32_t)w[j] == 1u) bq_push(q, slot, make_uint2((uint32_t)(v0 + i), (uint32_t)(w[j] >> 32)), F, ne);
                    }
                }
                bq_flush(q, slot, F, ne);
                slot ^= 1;
            }
        }
        if (b < nbins) {  // zero bin b (2^22-aligned: 16-byte stores)
            const uint64_t lo = (uint64_t)b << BIN_SHIFT, sz = min(nloc - lo, (uint64_t)1 << BIN_SHIFT);
            ulonglong2 *z = reinterpret_cast<ulonglong2 *>(state + lo);
            for (uint64_t i = tid; i < sz / 2; i += nthr) z[i] = make_ulonglong2(0ull, 0ull);
            if ((sz & 1) && tid == 0) state[lo + sz - 1] = 0ull;
        }
        grid.sync();
        if (b < nbins) {
            ull *st = state + ((uint64_t)b << BIN_SHIFT);
            const ull *ent = entries + base[b];
            const ull cnt = cursor[b];
            constexpr int RU = 8;
            for (ull i0 = tid; i0 < cnt; i0 += RU * nthr) {
                ull x[RU];
                #pragma unroll
                for (int u = 0; u < RU; u++) {
                    const ull i = i0 + (ull)u * nthr;
                    x[u] = i < cnt ? __ldcs(ent + i) : 0ull;
                }
                #pragma unroll
                for (int u = 0; u < RU; u++)
                    if (i0 + (ull)u * nthr < cnt) atomicAdd(st + (x[u] & mask), (x[u] & ~0xFFFFFFFFull) + 1ull);
            }
        }
        grid.sync();
    }
    block_add<256>(nf, removed);
}

template <int R>
static peel_status shard_build_r(const uint32_t *edges, uint64_t n, uint64_t m, uint64_t v0, uint64_t v1, ull *state,
                                 uint32_t *err, char *scratch, cudaStream_t s, bool *overflow, void *tmp,
                                 size_t tmp_bytes, const ShardF1 *f1) {
    const uint64_t nloc = v1 - v0;
    const ShardBins B = shard_bins(n, m, R, nloc);
    ull *cursor = (ull *)(scratch + B.cursor), *base = (ull *)(scratch + B.base), *cap = (ull *)(scratch + B.cap);
    uint32_t *flag = (uint32_t *)(scratch + B.flag);
    ull *entries = (ull *)(scratch + B.entries);
    *overflow = false;
    if (!f1) PEEL_CUDA(cudaMemsetAsync(state, 0, sizeof(ull) * nloc, s));  // f1: zeroed per bin, in L2
    PEEL_CUDA(cudaMemsetAsync(flag, 0, sizeof(uint32_t), s));
    {
        ProfScope ps("bin_init", s);
        bin_init_kernel<<<1, 32, 0, s>>>(n, nloc, m, R, B.nbins, cursor, base, cap);
    }
    const size_t smem = partition_smem(R, B.nbins);
    PEEL_CUDA(raise_smem((const void *)bin_partition_kernel<R>, smem));
    int pb = 0;
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pb, bin_partition_kernel<R>, PART_BLOCK, smem));
    if (pb < 1) pb = 1;
    int fpb = 0;
    if constexpr (R <= 5) PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fpb, shard_filter_kernel<R>, 256, 0));
    const SFGeom G = sf_geom(n, m, R, nloc, fpb);
    const char *sfe = getenv("PEEL_SHARD_FILTER");  // 0: bin_partition_kernel for every shard (A/B)
    // (R <= 5: the filter's staging is R 3 KB per warp of static shared memory)
    const bool filt = R <= 5 && m && tmp && G.bytes <= tmp_bytes && 4 * nloc <= n && !(sfe && atoi(sfe) == 0);
    uint32_t hflag = 0;
    if constexpr (R <= 5) if (filt) {
        SFHead *hd = (SFHead *)tmp;
        ull *counts = (ull *)((char *)tmp + sizeof(SFHead));
        ull *regions = (ull *)((char *)tmp + sizeof(SFHead) + al(sizeof(ull) * G.nblk));
        PEEL_CUDA(cudaMemsetAsync(hd, 0, sizeof(SFHead), s));
        {
            ProfScope ps("shard_filter", s);
            shard_filter_kernel<R><<<(unsigned)G.nblk, 256, 0, s>>>(edges, n, m, v0, v1, G.per_block, regions, G.cap_b,
                                                                   counts, err, &hd->ovf, ((uintptr_t)edges & 15) == 0);
        }
        const size_t bsm = shard_bin_smem(B.nbins);
        PEEL_CUDA(raise_smem((const void *)shard_bin_kernel, bsm));
        int bb = 0;
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bb, shard_bin_kernel, 256, bsm));
        {
            ProfScope ps("shard_bin", s);
            shard_bin_kernel<<<num_sms() * (bb < 1 ? 1 : bb), 256, bsm, s>>>(regions, G.cap_b, counts, G.nblk * G.cpr,
                                                                             G.cpr, (uint32_t)B.nbins, cursor, base,
                                                                             cap, entries, flag);
        }
        PEEL_CUDA(cudaGetLastError());
        uint32_t hovf = 0;
        PEEL_CUDA(cudaMemcpyAsync(&hovf, &hd->ovf, sizeof hovf, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof hflag, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaStreamSynchronize(s));
        if (hovf) {  // a region overflowed: the chunked partition from a clean slate
            PEEL_CUDA(cudaMemsetAsync(flag, 0, sizeof(uint32_t), s));
            bin_init_kernel<<<1, 32, 0, s>>>(n, nloc, m, R, B.nbins, cursor, base, cap);
        }
        if (!hovf) goto binned;
    }
    if (m) {
        ProfScope ps("bin_partition", s);
        bin_partition_kernel<R><<<num_sms() * pb, PART_BLOCK, smem, s>>>(edges, n, m, (uint32_t)B.nbins, cursor, base, cap,
                                                                          entries, err, flag, v0, v1, 0ull);
    }
    PEEL_CUDA(cudaGetLastError());
    PEEL_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof hflag, cudaMemcpyDeviceToHost, s));
    PEEL_CUDA(cudaStreamSynchronize(s));
binned:
    if (hflag) {
        *overflow = true;
        return PEEL_OK;
    }
    if (f1) {
        int per_sm = 0;
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, shard_accum_kernel, 256, 0));
        uint32_t nb = (uint32_t)B.nbins;
        uint32_t kk = f1->k;
        uint64_t nl = nloc, vv0 = v0;
        const ull *en = entries, *bs = base, *cu2 = cursor;
        ull *st = state, *pne = f1->ne, *pnf = f1->nf;
        uint2 *FF = (uint2 *)f1->F;
        void *args[] = {&en, &bs, &cu2, &nb, &nl, &vv0, &kk, &st, &FF, &pne, &pnf};
        ProfScope ps("shard_accum", s);
        PEEL_CUDA(cudaLaunchCooperativeKernel((void *)shard_accum_kernel, num_sms() * (per_sm < 1 ? 1 : per_sm), 256, args,
                                              0, s));
        return PEEL_OK;
    }
    uint64_t maxcap = 0;
    for (uint64_t b = 0; b < B.nbins; b++) maxcap = std::max<uint64_t>(maxcap, bin_capacity(n, nloc, m, R, b));
    const dim3 grid((unsigned)((maxcap + 256 * CSRB_PER - 1) / (256 * CSRB_PER)), (unsigned)B.nbins);
    if (m) {
        ProfScope ps("bin_red", s);
        bin_red_kernel<<<grid, 256, 0, s>>>(entries, base, cursor, state);
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}

ShardBinsView shard_bins_view(uint64_t n, uint64_t m, uint32_t r, uint64_t nloc, char *scratch) {
    const ShardBins B = shard_bins(n, m, r, nloc);
    ShardBinsView v;
    v.nbins = (uint32_t)B.nbins;
    v.cursor = (ull *)(scratch + B.cursor);
    v.base = (const ull *)(scratch + B.base);
    v.entries = (ull *)(scratch + B.entries);
    v.work = (ull *)(scratch + B.flag + 8);  // after the overflow flag, in the same 256-byte slot
    v.ctl = scratch + B.ctl;
    v.esort = (ull *)(scratch + B.esort);
    v.esort_words = (uint32_t)(2 * (((m + (1ull << EB_SHIFT) - 1) >> EB_SHIFT) + 1));
    return v;
}

// sort the shard's frontier entries (v, e) by edge bin into dst (see esort_scatter_kernel):
// the shard's kill phase then reads alive bits and rows per edge bin, from L2
peel_status shard_edge_sort(const void *src, const unsigned long long *pN, uint64_t nE_host, uint64_t m, void *dst,
                            const ShardBinsView &v, cudaStream_t s, bool zeroed) {
    if (!nE_host || !m) return PEEL_OK;
    const uint32_t enb = (uint32_t)((m + (1ull << EB_SHIFT) - 1) >> EB_SHIFT);
    ull *hist = v.esort, *cur = v.esort + enb + 1;
    const size_t essmem = esort_scatter_smem(enb);
    PEEL_CUDA(raise_smem((const void *)esort_scatter_kernel, essmem));
    if (!zeroed) PEEL_CUDA(cudaMemsetAsync(v.esort, 0, sizeof(ull) * 2 * (enb + 1), s));
    ProfScope ps("frontier_edge_sort", s);
    esort_hist_kernel<<<grid_for(nE_host, 8), 256, sizeof(uint32_t) * enb, s>>>((const uint2 *)src, pN, enb, hist);
    const uint64_t chunks = (nE_host + ES_CH - 1) / ES_CH;
    const unsigned sg = (unsigned)std::min<uint64_t>(chunks, (uint64_t)num_sms() * ES_BLOCKS);
    esort_scatter_kernel<<<sg ? sg : 1, 256, essmem, s>>>((const uint2 *)src, pN, enb, hist, cur, (uint2 *)dst);
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}

// phase D of a binned round on a shard: the decrements staged in the shard's bins (by
// dist.cu's kill/receive kernels) are applied by round_apply_kernel; crossings append
// (v0 + local id, remaining edge) to Fn.  |F_{t+1}| and Fn's length are copied to out_nf /
// out_ne (device words).
// the apply's counters zeroed before it, its |F_{t+1}| and entry count copied out after it: one
// tiny launch each instead of two memsets and two copies per shard and round
__global__ void shard_apply_prep_kernel(Ctl *ctl, ull *work) {
    const int i = threadIdx.x;
    if (i < (int)(sizeof(Ctl) / sizeof(ull))) reinterpret_cast<ull *>(ctl)[i] = 0ull;
    if (i == 0) *work = 0ull;
}
__global__ void shard_apply_post_kernel(const Ctl *ctl, uint32_t t, ull *out_nf, ull *out_ne) {
    *out_nf = ctl->nf[t % 3];
    *out_ne = ctl->ne[t % 3];
}

peel_status shard_apply(uint64_t nloc, uint64_t v0, uint32_t k, unsigned long long *state, void *Fn,
                        const ShardBinsView &v, uint32_t t, unsigned long long *out_nf, unsigned long long *out_ne,
                        cudaStream_t s) {
    static_assert(sizeof(Ctl) % sizeof(ull) == 0 && sizeof(Ctl) / sizeof(ull) <= 32, "Ctl zeroed by one warp");
    Ctl *ctl = (Ctl *)v.ctl;
    shard_apply_prep_kernel<<<1, 32, 0, s>>>(ctl, v.work);
    PeelArgs a;
    memset(&a, 0, sizeof a);
    a.n = nloc;
    a.k = k;
    a.state = state;
    a.F[0] = a.F[1] = Fn;
    a.ctl = ctl;
    a.v0 = v0;
    BinRound br;
    memset(&br, 0, sizeof br);
    br.nbins = v.nbins;
    br.cursor = v.cursor;
    br.base = v.base;
    br.entries = v.entries;
    br.work = v.work;
    br.t = t;
    const size_t dsmem = sizeof(uint32_t) * (v.nbins + 1);
    static thread_local std::map<std::pair<int, size_t>, int> dbc;  // (device, shared bytes) -> blocks per SM
    int dev = 0;
    PEEL_CUDA(cudaGetDevice(&dev));
    int &db = dbc[{dev, dsmem}];
    if (!db) {
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&db, round_apply_kernel, PEEL_BLOCK, dsmem));
        db = db < 1 ? 1 : db;
    }
    {
        ProfScope ps("round_apply", s);
        round_apply_kernel<<<num_sms() * db, PEEL_BLOCK, dsmem, s>>>(a, br);
    }
    shard_apply_post_kernel<<<1, 1, 0, s>>>(ctl, t, out_nf, out_ne);
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}

peel_status shard_build(uint32_t r, const uint32_t *edges, uint64_t n, uint64_t m, uint64_t v0, uint64_t v1,
                        unsigned long long *state, uint32_t *err, char *scratch, cudaStream_t s, bool *overflow,
                        void *tmp, size_t tmp_bytes, const ShardF1 *f1) {
    switch (r) {
        case 2: return shard_build_r<2>(edges, n, m, v0, v1, state, err, scratch, s, overflow, tmp, tmp_bytes, f1);
        case 3: return shard_build_r<3>(edges, n, m, v0, v1, state, err, scratch, s, overflow, tmp, tmp_bytes, f1);
        case 4: return shard_build_r<4>(edges, n, m, v0, v1, state, err, scratch, s, overflow, tmp, tmp_bytes, f1);
        case 5: return shard_build_r<5>(edges, n, m, v0, v1, state, err, scratch, s, overflow, tmp, tmp_bytes, f1);
        case 6: return shard_build_r<6>(edges, n, m, v0, v1, state, err, scratch, s, overflow, tmp, tmp_bytes, f1);
        case 7: return shard_build_r<7>(edges, n, m, v0, v1, state, err, scratch, s, overflow, tmp, tmp_bytes, f1);
        case 8: return shard_build_r<8>(edges, n, m, v0, v1, state, err, scratch, s, overflow, tmp, tmp_bytes, f1);
    }
    return PEEL_EINVAL;
}

}  // namespace peel

using namespace peel;

extern "C" size_t peel_kcore_workspace_bytes(uint64_t n, uint64_t m, uint32_t r, uint32_t k,
                                             uint32_t flags) {
    bool csr = use_csr(k, flags);
    if (!kcore_args_ok(n, m, r, csr)) return 0;
    return layout(n, m, r, csr).total;
}

static peel_status kcore_entry(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r, uint32_t k, uint32_t flags,
                               uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors, uint64_t *killed,
                               uint32_t cap, uint32_t *peel_round, void *workspace, size_t ws_bytes, void *stream,
                               const EdgeStream *es);

extern "C" peel_status peel_kcore(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r,
                                  uint32_t k, uint32_t flags, uint8_t *core_mask, uint32_t *rounds,
                                  uint64_t *survivors, uint64_t *killed, uint32_t cap,
                                  uint32_t *peel_round, void *workspace, size_t ws_bytes,
                                  void *stream) {
    return kcore_entry(edges, n, m, r, k, flags, core_mask, rounds, survivors, killed, cap, peel_round, workspace,
                       ws_bytes, stream, nullptr);
}

static peel_status kcore_entry(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r, uint32_t k, uint32_t flags,
                               uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors, uint64_t *killed,
                               uint32_t cap, uint32_t *peel_round, void *workspace, size_t ws_bytes, void *stream,
                               const EdgeStream *es) {
    bool csr = use_csr(k, flags);
    if (!kcore_args_ok(n, m, r, csr) || !rounds) return PEEL_EINVAL;
    if ((m && !edges) || (n && !core_mask) || !workspace) return PEEL_EINVAL;
    if ((flags & PEEL_FLAG_SUBROUNDS) && (csr || k > 2 || n % r != 0)) return PEEL_EINVAL;
    Layout L = layout(n, m, r, csr);
    if (ws_bytes < L.total) return PEEL_ENOMEM;
    prof_begin_call();
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        *rounds = 0;
        return PEEL_OK;
    }
    if (es && !m) es = nullptr;
    char *ws = (char *)workspace;
    switch (r) {
        case 2: return run_kcore<2>(edges, n, m, k, csr, flags, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s, es);
        case 3: return run_kcore<3>(edges, n, m, k, csr, flags, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s, es);
        case 4: return run_kcore<4>(edges, n, m, k, csr, flags, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s, es);
        case 5: return run_kcore<5>(edges, n, m, k, csr, flags, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s, es);
        case 6: return run_kcore<6>(edges, n, m, k, csr, flags, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s, es);
        case 7: return run_kcore<7>(edges, n, m, k, csr, flags, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s, es);
        case 8: return run_kcore<8>(edges, n, m, k, csr, flags, core_mask, rounds, survivors, killed, cap, peel_round, ws, L, s, es);
    }
    return PEEL_EINVAL;
}

extern "C" size_t peel_kcore_host_workspace_bytes(uint64_t n, uint64_t m, uint32_t r, uint32_t k,
                                                  uint32_t flags) {
    size_t w = peel_kcore_workspace_bytes(n, m, r, k, flags);
    if (!w) return 0;
    return w + al(sizeof(uint32_t) * r * m) + al(n) + 256;  // edges, mask, the mask's chunk flags
}

// The core mask back to the host (peel_kcore_host): the host buffer is zeroed by host threads
// while the GPU peels, and only the mask chunks that hold a core vertex are copied back -- none
// below the threshold, where the core is empty (C5: the 1 GB device-to-host copy, ~20 ms of the
// end-to-end step, is skipped).  Same bytes in the caller's buffer either way.
static constexpr uint32_t MASK_CHUNKS = 64;

__global__ void __launch_bounds__(256) mask_chunks_kernel(const uint8_t *__restrict__ mask, uint64_t n, uint64_t chunk,
                                                          uint32_t *flags) {
    const uint64_t n16 = n / 16;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * 256) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(mask) + i);
        if (v.x | v.y | v.z | v.w) flags[(i * 16) / chunk] = 1u;
    }
    for (uint64_t v = n16 * 16 + blockIdx.x * 256ull + threadIdx.x; v < n; v += (uint64_t)gridDim.x * 256)
        if (mask[v]) flags[v / chunk] = 1u;
}

struct HostZero {  // zero a host buffer on a few threads (joined by finish / the destructor)
    std::vector<std::thread> th;
    HostZero(uint8_t *p, uint64_t n) {
        const unsigned T = n >= (64ull << 20) ? 4u : (n ? 1u : 0u);
        for (unsigned t = 0; t < T; t++) {
            const uint64_t lo = n * t / T, hi = n * (t + 1) / T;
            th.emplace_back([=]() { memset(p + lo, 0, hi - lo); });
        }
    }
    void finish() {
        for (auto &x : th) x.join();
        th.clear();
    }
    ~HostZero() { finish(); }
};

static peel_status mask_to_host(const uint8_t *d_mask, uint8_t *h_mask, uint64_t n, uint32_t *d_flags, HostZero &hz,
                                cudaStream_t s) {
    if (!n) return PEEL_OK;
    const uint64_t chunk = (((n + MASK_CHUNKS - 1) / MASK_CHUNKS) + 15) & ~15ull;
    uint32_t hf[MASK_CHUNKS];
    PEEL_CUDA(cudaMemsetAsync(d_flags, 0, sizeof hf, s));
    {
        ProfScope ps("mask_chunks", s);
        mask_chunks_kernel<<<grid_for(n / 16 + 1), 256, 0, s>>>(d_mask, n, chunk, d_flags);
    }
    PEEL_CUDA(cudaGetLastError());
    PEEL_CUDA(cudaMemcpyAsync(hf, d_flags, sizeof hf, cudaMemcpyDeviceToHost, s));
    PEEL_CUDA(cudaStreamSynchronize(s));
    hz.finish();  // the zeros land before any chunk is copied over them
    for (uint32_t c = 0; c < MASK_CHUNKS; c++) {
        const uint64_t lo = c * chunk;
        if (!hf[c] || lo >= n) continue;
        const uint64_t len = std::min<uint64_t>(chunk, n - lo);
        PEEL_CUDA(cudaMemcpyAsync(h_mask + lo, d_mask + lo, len, cudaMemcpyDeviceToHost, s));
    }
    PEEL_CUDA(cudaStreamSynchronize(s));
    return PEEL_OK;
}

extern "C" peel_status peel_kcore_host(const uint32_t *edges_host, uint64_t n, uint64_t m,
                                       uint32_t r, uint32_t k, uint32_t flags,
                                       uint8_t *core_mask_host, uint32_t *rounds,
                                       uint64_t *survivors, uint64_t *killed, uint32_t cap,
                                       void *workspace, size_t ws_bytes, void *stream) {
    size_t w = peel_kcore_workspace_bytes(n, m, r, k, flags);
    if (!w || !rounds || !workspace || (m && !edges_host) || (n && !core_mask_host)) return PEEL_EINVAL;
    if (ws_bytes < peel_kcore_host_workspace_bytes(n, m, r, k, flags)) return PEEL_ENOMEM;
    cudaStream_t s = (cudaStream_t)stream;
    char *base = (char *)workspace;
    uint32_t *d_edges = (uint32_t *)(base + w);
    uint8_t *d_mask = (uint8_t *)(base + w + al(sizeof(uint32_t) * r * m));
    // binned builds: the copy runs on a second stream in 16 chunks, and the build partitions
    // each chunk as it lands (the copy stream first waits for work already queued on s).
    // Other paths (and small inputs, where the extra stream costs more than it hides): one copy.
    if (use_csr(k, flags) || n <= BIN_MIN_N || (flags & PEEL_FLAG_SUBROUNDS)) {
        if (m) PEEL_CUDA(cudaMemcpyAsync(d_edges, edges_host, sizeof(uint32_t) * r * m, cudaMemcpyHostToDevice, s));
        peel_status st = peel_kcore(d_edges, n, m, r, k, flags, d_mask, rounds, survivors, killed, cap, nullptr,
                                    workspace, w, stream);
        if (st != PEEL_OK && st != PEEL_ETRUNC) return st;
        if (n) PEEL_CUDA(cudaMemcpyAsync(core_mask_host, d_mask, n, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaStreamSynchronize(s));
        return st;
    }
    // per host thread and device: concurrent calls (distinct streams and workspaces, peel.h)
    // each get their own copy stream and events, and no lock is held across the peel
    HostZero hz(core_mask_host, n);
    static thread_local std::map<int, std::pair<cudaStream_t, std::vector<cudaEvent_t>>> res;
    int dev = 0;
    PEEL_CUDA(cudaGetDevice(&dev));
    auto &rs = res[dev];
    if (!rs.first) {
        PEEL_CUDA(cudaStreamCreateWithFlags(&rs.first, cudaStreamNonBlocking));
        rs.second.resize(17);
        for (auto &e : rs.second) PEEL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    EdgeStream es;
    es.host = edges_host;
    es.dev = d_edges;
    es.copy = rs.first;
    const uint64_t nchunks = m ? std::min<uint64_t>(16, m) : 0;
    es.chunk = nchunks ? (m + nchunks - 1) / nchunks : 1;
    es.done.assign(rs.second.begin(), rs.second.begin() + (nchunks ? (m + es.chunk - 1) / es.chunk : 0));
    if (m) {
        PEEL_CUDA(cudaEventRecord(rs.second[16], s));
        PEEL_CUDA(cudaStreamWaitEvent(es.copy, rs.second[16], 0));
    }
    peel_status st = kcore_entry(d_edges, n, m, r, k, flags, d_mask, rounds, survivors, killed, cap, nullptr,
                                 workspace, w, stream, m ? &es : nullptr);
    if (st != PEEL_OK && st != PEEL_ETRUNC) return st;
    const peel_status sm = mask_to_host(d_mask, core_mask_host, n, (uint32_t *)(base + w + al(sizeof(uint32_t) * r * m) + al(n)), hz, s);
    return sm != PEEL_OK ? sm : st;
}
