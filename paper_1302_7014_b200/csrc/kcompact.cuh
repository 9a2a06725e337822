// kcompact.cuh -- the binned rounds of the packed (k <= 2) path for n > 2^23 (part of
// kcore.cu; included after its binned-round kernels; DESIGN.md §5 "Slot-compacted rounds").
//
// The schedule is kcore.cu's (F_t = alive vertices of degree < k, all removed with
// their alive edges, until F_t is empty), with the same crossing rule: the ONE decrement that
// takes a count from k to k-1 puts the vertex in F_{t+1} with the entry (v, id sum - e), its
// one alive edge.  What changes is where the state lives and how the frontier is ordered.
//
//   slots      the state of vertex v lives in a SLOT.  Until the first compaction the slots are
//              the identity (state[v], kcore.cu's array).  When the live set L (count >= k)
//              has halved since the slots were laid out, a compaction pass copies the live
//              states densely, bin by bin (2^22 vertices), to [b 2^22, b 2^22 + |L ∩ b|) of a
//              compact buffer, and writes a record per 64-vertex group {slot mask, index of its
//              first slot}: slot(v) = base + popc(mask & below(v)).  Between compactions a
//              vertex that leaves keeps its slot (its count < k never matches the crossing test
//              again: a frontier vertex gets at most one more decrement, a dead one none).
//   build      kcore.cu's binned build (partition, then per-bin L2-resident accumulation); the
//              scan of each bin emits F_1's entries (v, id sum) straight into per-EDGE-bin
//              regions -- the kill phase's input order (no separate sort pass).
//   round t    kill: F_t in edge-bin order; exactly-once kill (alive test-and-clear); the
//              killed edges' decrements partitioned by vertex bin (round_kill_partition's body).
//              apply: per vertex bin in order, each decrement finds its vertex's slot (a
//              record lookup once compacted) and applies a returning 64-bit atomic; a crossing
//              stages its entry in shared memory, sorted into the edge-bin regions.  The bin
//              after next has its slots (and records) prefetched into L2: a round streams the
//              SLOT count, <= 2 |L| after the first compaction, instead of the whole n.
//   end        core_mask[v] = count(slot(v)) >= k (0 without a slot).  A tail with a large live
//              set and a small frontier (above threshold) hands over to kcore.cu's persistent
//              kernel, after writing the slots back to the full state array when compacted.

struct __align__(16) CRec {
    ull mask;       // bit i: vertex 64 g + i has a slot
    uint32_t base;  // slot of its first vertex with a slot (absolute index)
    uint32_t pad;
};
static_assert(sizeof(CRec) == 16, "16-byte group record");

static constexpr int CB_BLOCK = 256;
static constexpr int GB = 4;         // compaction: groups per batch (registers: 2 GB states per lane)
static constexpr int CGW = 32;       // compaction: groups per warp per item (8 CGW per block item)
#ifndef PEEL_FE_CAP_A
#define PEEL_FE_CAP_A 2048
#endif
#ifndef PEEL_FE_CAP_B
#define PEEL_FE_CAP_B 2048
#endif
static constexpr int FE_CAP_A = PEEL_FE_CAP_A;  // apply: frontier entries staged per block before an edge-bin sort
static constexpr int FE_CAP_B = PEEL_FE_CAP_B;  // build scan (F_1 is ~24% of n: longer runs per edge bin)
// the kill: 4 entries per thread at 4 resident blocks per SM (C5 kill 25.0 -> 24.0 ms against
// round 1's 3 at 5, which kcore.cu's uncompacted kill keeps)
#ifndef PEEL_CKU
#define PEEL_CKU 4
#endif
#ifndef PEEL_CKILL_MINB
#define PEEL_CKILL_MINB 4
#endif
// the apply prefetches the entries of the item one wave (gridDim.x items) ahead into L2:
// C5 apply 23.91 -> 23.69 ms.  (The kill's rows prefetched before the alive test: 24.15 ->
// 25.31 ms, removed: the losing entries' lines cost more than the overlap saves.)
#ifndef PEEL_CAPPLY_PF
#define PEEL_CAPPLY_PF 1
#endif
static constexpr int CKU = PEEL_CKU;
static constexpr int CKCH = PART_BLOCK * CKU;
#ifndef PEEL_CB_RU
#define PEEL_CB_RU 8
#endif
#ifndef PEEL_CB_SU
#define PEEL_CB_SU 4
#endif
#ifndef PEEL_CDCH
#define PEEL_CDCH 512
#endif
static constexpr int CDCH = PEEL_CDCH;  // apply: decrement entries per work item

__host__ __device__ inline uint64_t bin_groups(uint64_t n, uint64_t b) { return (bin_size(n, b) + 63) >> 6; }

// Device-side round control (the rounds run without a host sync each: see run_compact).  One
// thread of cround_ctl_kernel decides, before every round, whether the peel is done, whether
// the tail goes to the persistent kernel or the slots are due for compaction (the host's
// work), or the round runs -- then zeroes the round's counters.  Every round kernel exits at
// once when `stop` is set.
enum : uint32_t { RC_RUN = 0, RC_DONE = 1, RC_TAIL = 2, RC_COMPACT = 3 };
struct RoundCtl {
    uint32_t t;       // the round to run next
    uint32_t stop;    // RC_*
    uint32_t ran;     // the round t was launched (t advances at the next decision)
    uint32_t live_t;  // the round whose |F_t| was last taken off `live`
    ull live;         // vertices with count >= k after the last completed round
    ull nslots;       // slots laid out
};
struct RoundRule {    // the thresholds (compact_at, ctail_live_frac, ctail_ratio)
    uint64_t n;
    double frac, tail, tratio, at, at1;  // at1: the first compaction (identity slots)
    int compaction;
};

struct CArgs {
    const uint32_t *edges;
    uint64_t n, m;
    uint32_t k, t;           // t: the round (apply: emits F_{t+1}; build: t = 0 emits F_1)
    uint32_t nbins, enb;
    ull *X;                  // slots this round (identity: the full state array)
    ull *Y;                  // compaction: the new slots
    CRec *recs;              // [ceil(n / 64)] (compacted slots)
    ull *alloc;              // compaction: [nbins] new slots per bin (allocation cursor)
    const ull *slots;        // [nbins] slots per bin (prefetch length), compacted
    uint2 *fe;               // frontier regions: edge bin j at j fe_stride
    uint64_t fe_stride;
    ull *fecnt;              // [enb] entries written per edge bin (F_{t+1})
    const ull *fecur;        // [enb] entries of F_t per edge bin
    Ctl *ctl;
    ull *stats;
    uint32_t stat_cap;
    uint32_t *peel_round;
    const ull *cursor;       // decrement bins (kcore.cu's entry buffer)
    const ull *base;
    const ull *entries;
    ull *work;
    ull *live_total;         // build: vertices with count >= k
    RoundCtl *rc;            // rounds: the round index and the stop flag (device-side loop)
    ull *fec[2];             // rounds: per-edge-bin entry counts by round parity
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// exclusive prefix of cnt[0 .. ns) into pre[0 .. ns] (shared memory, ns <= 32 K); every thread
// of the block calls it after writing cnt = pre (in place)
__device__ __forceinline__ void block_excl_scan(uint32_t *pre, uint32_t ns) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint32_t per = (ns + 31) / 32;
        uint32_t loc = 0;
        for (uint32_t q = 0; q < per; q++) {
            const uint32_t i = threadIdx.x * per + q;
            loc += i < ns ? pre[i] : 0;
        }
        uint32_t x = loc;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if ((int)threadIdx.x >= o) x += y;
        }
        uint32_t run = x - loc;
        for (uint32_t q = 0; q < per; q++) {
            const uint32_t i = threadIdx.x * per + q;
            if (i < ns) { const uint32_t c = pre[i]; pre[i] = run; run += c; }
        }
        if (threadIdx.x == 31) pre[ns] = x;
    }
    __syncthreads();
}

// ---- frontier staging: entries (v, e) counting-sorted by edge bin e >> EB_SHIFT in shared
// memory and written as one run per bin into that bin's region.  Dynamic shared memory:
// buf[FE_CAP] uint2, gpos[enb] u64, hist[enb] u32, offs[enb] u32.
struct FeView {
    uint2 *buf;
    ull *gpos;
    uint32_t *hist, *offs;
    uint32_t *n;   // staged entries
    ull *fecnt;    // the regions' entry counts being written (F_{t+1})
};

template <int CAP>
__device__ __forceinline__ FeView fe_view(unsigned char *smem, uint32_t enb, uint32_t *n, ull *fecnt) {
    FeView f;
    f.fecnt = fecnt;
    f.buf = (uint2 *)smem;
    f.gpos = (ull *)(f.buf + CAP);
    f.hist = (uint32_t *)(f.gpos + enb);
    f.offs = f.hist + enb;
    f.n = n;
    return f;
}

static size_t fe_smem(int cap, uint32_t enb) { return sizeof(uint2) * cap + (sizeof(ull) + 2 * sizeof(uint32_t)) * enb; }

// warp-aggregated push; past CAP the entry goes straight to its region (one global atomic)
template <int CAP>
__device__ __forceinline__ void fe_push(const FeView &f, const CArgs &a, uint2 v) {
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t pos = 0;
    if (g.thread_rank() == 0) pos = atomicAdd(f.n, (uint32_t)g.size());
    pos = g.shfl(pos, 0) + g.thread_rank();
    if (pos < CAP) {
        f.buf[pos] = v;
    } else {
        const uint32_t j = v.y >> EB_SHIFT;
        const ull p = atomicAdd(f.fecnt + j, 1ull);
        a.fe[(ull)j * a.fe_stride + p] = v;
    }
}

// every thread of the block calls it
template <int CAP>
__device__ void fe_flush(const FeView &f, const CArgs &a) {
    constexpr int PER = CAP / CB_BLOCK;
    __syncthreads();
    const uint32_t cnt = min(*f.n, (uint32_t)CAP);
    if (cnt == 0) return;  // uniform: every thread read the same count after the barrier
    for (uint32_t j = threadIdx.x; j < a.enb; j += CB_BLOCK) f.hist[j] = 0;
    __syncthreads();
    uint2 v[PER];
    uint32_t rk[PER];
    #pragma unroll
    for (int q = 0; q < PER; q++) {
        const uint32_t i = q * CB_BLOCK + threadIdx.x;
        if (i < cnt) {
            v[q] = f.buf[i];
            rk[q] = atomicAdd(&f.hist[v[q].y >> EB_SHIFT], 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of hist (enb <= 1024): one warp
        const uint32_t per = (a.enb + 31) / 32;
        uint32_t loc = 0;
        for (uint32_t q = 0; q < per; q++) {
            const uint32_t j = threadIdx.x * per + q;
            loc += j < a.enb ? f.hist[j] : 0;
        }
        uint32_t x = loc;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if ((int)threadIdx.x >= o) x += y;
        }
        uint32_t run = x - loc;
        for (uint32_t q = 0; q < per; q++) {
            const uint32_t j = threadIdx.x * per + q;
            if (j < a.enb) { f.offs[j] = run; run += f.hist[j]; }
        }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < a.enb; j += CB_BLOCK)
        if (f.hist[j]) f.gpos[j] = atomicAdd(f.fecnt + j, (ull)f.hist[j]);
    #pragma unroll
    for (int q = 0; q < PER; q++) {
        const uint32_t i = q * CB_BLOCK + threadIdx.x;
        if (i < cnt) f.buf[f.offs[v[q].y >> EB_SHIFT] + rk[q]] = v[q];
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += CB_BLOCK) {
        const uint2 x = f.buf[i];
        const uint32_t j = x.y >> EB_SHIFT;
        a.fe[(ull)j * a.fe_stride + f.gpos[j] + (i - f.offs[j])] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) *f.n = 0;
    __syncthreads();
}

// ---- one compaction item: 8 CGW 64-vertex groups of bin b starting at group g0 (global id),
// warp w taking CGW of them, lane = vertex within the group.  IDENT: the source slots are the
// identity (src = the full state array); else the records' slots in src.  Two passes: count
// the vertices that stay live (count >= k), one allocation per item, then write them densely
// and the new records.  Every thread of the block calls it.
template <bool IDENT>
__device__ void compact_item(const CArgs &a, uint32_t b, uint64_t g0, const ull *src, uint32_t *wsh) {
    static_assert(CGW % GB == 0 && CGW <= 32, "batches of GB groups, one record per lane");
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gbin0 = (uint64_t)b << (BIN_SHIFT - 6);
    const uint64_t gend = gbin0 + bin_groups(a.n, b);  // this bin's groups
    const uint64_t gw0 = g0 + (uint64_t)w * CGW;
    const uint32_t k = a.k;
    // lane l: the record of group gw0 + l
    ull mymask = 0;
    uint32_t mybase = 0;
    {
        const uint64_t g = gw0 + lane;
        if (lane < CGW && g < gend) {
            if (IDENT) {
                const uint64_t v0 = g << 6;
                const uint64_t nv = min((uint64_t)64, a.n - v0);
                mymask = nv == 64 ? ~0ull : ((1ull << nv) - 1);
                mybase = (uint32_t)v0;
            } else {
                const uint4 r = __ldcg(reinterpret_cast<const uint4 *>(a.recs + g));
                mymask = ((ull)r.y << 32) | r.x;
                mybase = r.z;
            }
        }
    }
    // a warp whose groups have no slot left has nothing to copy and no record to change
    const bool any = __ballot_sync(0xffffffffu, mymask != 0ull) != 0u;
    // pass 1: vertices that stay, per warp
    uint32_t keepcnt = 0;
    #pragma unroll 2
    for (int i = 0; i < (any ? CGW / GB : 0); i++) {
        ull st[GB][2];
        ull mk[GB];
        #pragma unroll
        for (int j = 0; j < GB; j++) {
            const ull m = __shfl_sync(0xffffffffu, mymask, GB * i + j);
            const uint32_t bs = __shfl_sync(0xffffffffu, mybase, GB * i + j);
            mk[j] = m;
            #pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t bit = 32 * h + lane;
                const bool has = (m >> bit) & 1ull;
                st[j][h] = has ? __ldca(src + bs + __popcll(m & ((1ull << bit) - 1ull))) : 0ull;
            }
        }
        #pragma unroll
        for (int j = 0; j < GB; j++)
            #pragma unroll
            for (int h = 0; h < 2; h++) {
                const bool keep = ((mk[j] >> (32 * h + lane)) & 1ull) && (uint32_t)st[j][h] >= k;
                keepcnt += __popc(__ballot_sync(0xffffffffu, keep));
            }
    }
    if (lane == 0) wsh[w] = keepcnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int q = 0; q < CB_BLOCK / 32; q++) { const uint32_t c = wsh[q]; wsh[q] = tot; tot += c; }
        const ull base = tot ? atomicAdd(a.alloc + b, (ull)tot) : 0ull;
        wsh[CB_BLOCK / 32] = (uint32_t)(((uint64_t)b << BIN_SHIFT) + base);
    }
    __syncthreads();
    uint32_t run = wsh[CB_BLOCK / 32] + wsh[w];
    // pass 2: the same states again (L1 / L2 hits), written densely, new records
    #pragma unroll 2
    for (int i = 0; i < (any ? CGW / GB : 0); i++) {
        ull st[GB][2];
        ull mk[GB];
        #pragma unroll
        for (int j = 0; j < GB; j++) {
            const ull m = __shfl_sync(0xffffffffu, mymask, GB * i + j);
            const uint32_t bs = __shfl_sync(0xffffffffu, mybase, GB * i + j);
            mk[j] = m;
            #pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t bit = 32 * h + lane;
                const bool has = (m >> bit) & 1ull;
                st[j][h] = has ? __ldca(src + bs + __popcll(m & ((1ull << bit) - 1ull))) : 0ull;
            }
        }
        ull nm = 0;
        uint32_t nb = 0;
        #pragma unroll
        for (int j = 0; j < GB; j++) {
            const bool k0 = ((mk[j] >> lane) & 1ull) && (uint32_t)st[j][0] >= k;
            const bool k1 = ((mk[j] >> (32 + lane)) & 1ull) && (uint32_t)st[j][1] >= k;
            const uint32_t b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
            if (k0) a.Y[run + __popc(b0 & lanemask_lt())] = st[j][0];
            if (k1) a.Y[run + __popc(b0) + __popc(b1 & lanemask_lt())] = st[j][1];
            if (lane == j) { nm = ((ull)b1 << 32) | b0; nb = run; }
            run += __popc(b0) + __popc(b1);
        }
        const uint64_t g = gw0 + GB * i + lane;
        if (lane < GB && g < gend)
            __stcg(reinterpret_cast<uint4 *>(a.recs + g), make_uint4((uint32_t)nm, (uint32_t)(nm >> 32), nb, 0u));
    }
}

// compaction pass over every bin (non-cooperative; items handed out by a counter in bin order)
// the same with the item's states held in registers (8 groups per warp, 16 states per lane):
// one load pass, no reload after the allocation (PEEL_CREG, default)
static constexpr int CRG = 8;
template <bool IDENT>
__device__ void compact_item_reg(const CArgs &a, uint32_t b, uint64_t g0, const ull *src, uint32_t *wsh) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gend = ((uint64_t)b << (BIN_SHIFT - 6)) + bin_groups(a.n, b);
    const uint64_t gw0 = g0 + (uint64_t)w * CRG;
    const uint32_t k = a.k;
    ull mymask = 0;
    uint32_t mybase = 0;
    {
        const uint64_t g = gw0 + lane;
        if (lane < CRG && g < gend) {
            if (IDENT) {
                const uint64_t v0 = g << 6;
                const uint64_t nv = min((uint64_t)64, a.n - v0);
                mymask = nv == 64 ? ~0ull : ((1ull << nv) - 1);
                mybase = (uint32_t)v0;
            } else {
                const uint4 r = __ldcg(reinterpret_cast<const uint4 *>(a.recs + g));
                mymask = ((ull)r.y << 32) | r.x;
                mybase = r.z;
            }
        }
    }
    ull st[CRG][2];
    #pragma unroll
    for (int j = 0; j < CRG; j++) {
        const ull m = __shfl_sync(0xffffffffu, mymask, j);
        const uint32_t bs = __shfl_sync(0xffffffffu, mybase, j);
        #pragma unroll
        for (int h = 0; h < 2; h++) {
            const uint32_t bit = 32 * h + lane;
            const bool has = (m >> bit) & 1ull;
            // a state that stays has count >= k >= 1; 0 marks "no slot"
            st[j][h] = has ? __ldcs(src + bs + __popcll(m & ((1ull << bit) - 1ull))) : 0ull;
        }
    }
    uint32_t keepcnt = 0;
    #pragma unroll
    for (int j = 0; j < CRG; j++)
        #pragma unroll
        for (int h = 0; h < 2; h++) keepcnt += __popc(__ballot_sync(0xffffffffu, (uint32_t)st[j][h] >= k && st[j][h]));
    if (lane == 0) wsh[w] = keepcnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int q = 0; q < CB_BLOCK / 32; q++) { const uint32_t c = wsh[q]; wsh[q] = tot; tot += c; }
        const ull base = tot ? atomicAdd(a.alloc + b, (ull)tot) : 0ull;
        wsh[CB_BLOCK / 32] = (uint32_t)(((uint64_t)b << BIN_SHIFT) + base);
    }
    __syncthreads();
    uint32_t run = wsh[CB_BLOCK / 32] + wsh[w];
    #pragma unroll
    for (int j = 0; j < CRG; j++) {
        const bool k0 = st[j][0] && (uint32_t)st[j][0] >= k, k1 = st[j][1] && (uint32_t)st[j][1] >= k;
        const uint32_t b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
        if (k0) a.Y[run + __popc(b0 & lanemask_lt())] = st[j][0];
        if (k1) a.Y[run + __popc(b0) + __popc(b1 & lanemask_lt())] = st[j][1];
        const uint64_t g = gw0 + j;
        const ull mj = __shfl_sync(0xffffffffu, mymask, j);  // every lane: a shuffle is warp-wide
        if (lane == 0 && g < gend && (mj || b0 || b1))
            __stcg(reinterpret_cast<uint4 *>(a.recs + g), make_uint4(b0, b1, run, 0u));
        run += __popc(b0) + __popc(b1);
    }
}

template <bool IDENT>
__global__ void __launch_bounds__(CB_BLOCK, 4) ccompact_reg_kernel(CArgs a) {
    __shared__ uint32_t wsh[CB_BLOCK / 32 + 1];
    __shared__ ull item[2];
    const uint64_t per_bin = (1ull << (BIN_SHIFT - 6)) / (8 * CRG);  // items of a full bin
    const uint64_t nitems = (uint64_t)a.nbins * per_bin;
    for (int ib = 0;; ib ^= 1) {
        if (threadIdx.x == 0) item[ib] = atomicAdd(a.work, 1ull);
        __syncthreads();
        const ull c = item[ib];
        if (c >= nitems) break;
        const uint32_t b = (uint32_t)(c / per_bin);
        const uint64_t g0 = ((uint64_t)b << (BIN_SHIFT - 6)) + (c % per_bin) * 8 * CRG;
        if (g0 < ((uint64_t)b << (BIN_SHIFT - 6)) + bin_groups(a.n, b)) compact_item_reg<IDENT>(a, b, g0, a.X, wsh);
        __syncthreads();  // wsh is rewritten next item
    }
}

template <bool IDENT>
__global__ void __launch_bounds__(CB_BLOCK, 4) ccompact_kernel(CArgs a) {
    __shared__ uint32_t wsh[CB_BLOCK / 32 + 1];
    __shared__ ull item;
    const uint64_t per_bin = ((1ull << (BIN_SHIFT - 6)) + 8 * CGW - 1) / (8 * CGW);  // items of a full bin
    const uint64_t nitems = (((a.n + 63) >> 6) + 8 * CGW - 1) / (8 * CGW);
    for (;;) {
        if (threadIdx.x == 0) item = atomicAdd(a.work, 1ull);
        __syncthreads();
        const ull c = item;
        if (c >= nitems) break;
        const uint32_t b = (uint32_t)(c / per_bin);
        const uint64_t g0 = ((uint64_t)b << (BIN_SHIFT - 6)) + (c % per_bin) * 8 * CGW;
        if (g0 < ((uint64_t)b << (BIN_SHIFT - 6)) + bin_groups(a.n, b)) compact_item<IDENT>(a, b, g0, a.X, wsh);
        __syncthreads();  // item and wsh are rewritten next iteration
    }
}

// ---- build: kcore.cu's binned accumulation (cooperative: zero bin b, grid barrier, its
// entries as L2-resident REDs, grid barrier), the scan of each bin emitting F_1 -- the
// count-1 vertices' entries (v, id sum) -- into the edge-bin regions while the bin is in L2.
template <int R>
__global__ void __launch_bounds__(CB_BLOCK, 4) cbuild_kernel(CArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t fen;
    if (threadIdx.x == 0) fen = 0;
    __syncthreads();
    const FeView f = fe_view<FE_CAP_B>(smem_raw, a.enb, &fen, a.fecnt);
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const ull mask = (1ull << BIN_SHIFT) - 1;
    constexpr int SU = PEEL_CB_SU;  // states per thread per scan step
    ull leavers = 0, emitted = 0, kept = 0;
    auto scan_bin = [&](uint32_t sb) {  // bin sb's states (in L2): F_1 entries, leavers, survivors
        const uint64_t lo = (uint64_t)sb << BIN_SHIFT, hi = lo + bin_size(a.n, sb);
        for (uint64_t base = lo + (uint64_t)blockIdx.x * CB_BLOCK * SU; base < hi;
             base += (uint64_t)gridDim.x * CB_BLOCK * SU) {
            ull w[SU];
            #pragma unroll
            for (int j = 0; j < SU; j++) {
                const uint64_t v = base + (uint64_t)j * CB_BLOCK + threadIdx.x;
                w[j] = v < hi ? __ldcg(a.X + v) : ~0ull;
            }
            #pragma unroll
            for (int j = 0; j < SU; j++) {
                const uint64_t v = base + (uint64_t)j * CB_BLOCK + threadIdx.x;
                if (v >= hi) continue;
                const uint32_t c = (uint32_t)w[j];
                if (c >= a.k) { kept++; continue; }
                leavers++;
                if (a.peel_round) a.peel_round[v] = 1;
                if (c == 1u) {  // k = 2: its one edge is the id sum
                    emitted++;
                    fe_push<FE_CAP_B>(f, a, make_uint2((uint32_t)v, (uint32_t)(w[j] >> 32)));
                }
            }
            __syncthreads();  // every push of this step landed: one decision for the block
            if (fen >= FE_CAP_B - CB_BLOCK * SU) fe_flush<FE_CAP_B>(f, a);
            __syncthreads();
        }
    };
    auto zero_bin = [&](uint32_t zb) {
        const uint64_t lo = (uint64_t)zb << BIN_SHIFT, sz = bin_size(a.n, zb);
        ulonglong2 *z = reinterpret_cast<ulonglong2 *>(a.X + lo);  // lo is 2^22-aligned
        for (uint64_t i = tid; i < sz / 2; i += nthr) z[i] = make_ulonglong2(0ull, 0ull);
        if ((sz & 1) && tid == 0) a.X[lo + sz - 1] = 0ull;
    };
    auto red_bin = [&](uint32_t rb) {
        // RU entry loads in flight per thread before their REDs (one load at a time left the
        // loop waiting on DRAM latency: the load -> RED dependency was ncu's top stall)
        constexpr int RU = PEEL_CB_RU;
        ull *st = a.X + ((uint64_t)rb << BIN_SHIFT);
        const ull *ent = a.entries + a.base[rb];
        const ull cnt = a.cursor[rb];
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
    };
    for (uint32_t b = 0; b <= a.nbins; b++) {
        if (b > 0) scan_bin(b - 1);  // bin b-1 (still in L2), overlapped with zeroing bin b
        if (b < a.nbins) zero_bin(b);
        grid.sync();
        if (b < a.nbins) red_bin(b);
        grid.sync();
    }
    fe_flush<FE_CAP_B>(f, a);
    block_add<CB_BLOCK>(&a.ctl->nf[0], leavers);
    block_add<CB_BLOCK>(&a.ctl->ne[0], emitted);
    block_add<CB_BLOCK>(a.live_total, kept);
}

// ---- kill: F_t's entries read from the edge-bin regions in bin order (round_kill_partition's
// body; the decrements are partitioned by vertex bin into the entry buffer)
template <int R>
__global__ void __launch_bounds__(PART_BLOCK, PEEL_CKILL_MINB) ckill_kernel(PeelArgs a, BinRound br, CArgs c) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t nbins = br.nbins;
    ull *sorted = (ull *)smem_raw;                       // [(R-1) CKCH] the chunk's decrements, bin-sorted
    ull *gpos = sorted + (R - 1) * CKCH;                  // [nbins]
    uint32_t *hist = (uint32_t *)(gpos + nbins);         // [nbins]
    uint32_t *offs = hist + nbins;                       // [nbins]
    uint32_t *pre = offs + nbins;                        // [enb + 1] chunks before edge bin j
    __shared__ uint32_t total;
    Ctl *ctl = a.ctl;
    if (c.rc && *(volatile uint32_t *)&c.rc->stop) return;  // uniform: the loop stopped before this round
    const uint32_t t = c.rc ? *(volatile uint32_t *)&c.rc->t : br.t;
    const ull *fecur = c.rc ? (((t - 1) & 1) ? c.fec[1] : c.fec[0]) : c.fecur;
    for (uint32_t j = threadIdx.x; j < c.enb; j += PART_BLOCK)
        pre[j] = (uint32_t)((ld_cg_u64(fecur + j) + CKCH - 1) / CKCH);
    block_excl_scan(pre, c.enb);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (t <= a.stat_cap) a.rtime[t - 1] = globaltimer();
        a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap)] = ld_cg_u64(&ctl->nf[(t - 1) % 3]);
        ctl->nf[(t + 1) % 3] = 0;
        ctl->ne[(t + 1) % 3] = 0;
    }
    __syncthreads();
    __syncthreads();
    const uint32_t nitems = pre[c.enb];
    const ull mask = (1ull << BIN_SHIFT) - 1;
    ull kills = 0;
    for (uint32_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        uint32_t lo = 0, hi = c.enb;  // edge bin j with pre[j] <= item < pre[j+1]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= item) lo = mid; else hi = mid;
        }
        const ull off = (ull)(item - pre[lo]) * CKCH;
        const ull nE = min((ull)CKCH, ld_cg_u64(fecur + lo) - off);
        const uint2 *Fc = c.fe + (ull)lo * c.fe_stride + off;
        uint2 ent[CKU];
        bool win[CKU];
        #pragma unroll
        for (int q = 0; q < CKU; q++) {
            const uint32_t i = q * PART_BLOCK + threadIdx.x;
            ent[q] = i < nE ? __ldcg(Fc + i) : make_uint2(0u, 0u);
        }
        for (uint32_t b = threadIdx.x; b < nbins; b += PART_BLOCK) hist[b] = 0;
        uint32_t oldw[CKU];
        #pragma unroll
        for (int q = 0; q < CKU; q++) {
            const uint32_t i = q * PART_BLOCK + threadIdx.x;
            oldw[q] = 0;
            if (i < nE) oldw[q] = atomicAnd(a.alive + (ent[q].y >> 5), ~(1u << (ent[q].y & 31)));
        }
        uint32_t ue[CKU][R];
        #pragma unroll
        for (int q = 0; q < CKU; q++) {
            const uint32_t i = q * PART_BLOCK + threadIdx.x;
            win[q] = i < nE && ((oldw[q] >> (ent[q].y & 31)) & 1u);
            if (win[q]) load_row<R>(a.edges, ent[q].y, a.m, a.edges_vec, ue[q]);
            kills += win[q];
        }
        __syncthreads();  // hist zeroed
        uint32_t rk[CKU][R];
        #pragma unroll
        for (int q = 0; q < CKU; q++)
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (win[q] && ue[q][r] != ent[q].x) rk[q][r] = atomicAdd(&hist[ue[q][r] >> BIN_SHIFT], 1u);
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
        for (uint32_t b = threadIdx.x; b < nbins; b += PART_BLOCK)  // absolute run starts
            if (hist[b]) gpos[b] = br.base[b] + atomicAdd(br.cursor + b, (ull)hist[b]);
        #pragma unroll
        for (int q = 0; q < CKU; q++)
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (win[q] && ue[q][r] != ent[q].x)
                    sorted[offs[ue[q][r] >> BIN_SHIFT] + rk[q][r]] = ((ull)ent[q].y << 32) | ue[q][r];
        __syncthreads();
        const uint32_t tot = total;
        for (uint32_t i = threadIdx.x; i < tot; i += PART_BLOCK) {
            const ull v = sorted[i];
            const uint32_t b = (uint32_t)v >> BIN_SHIFT;
            br.entries[gpos[b] + (i - offs[b])] = v & ~(0xFFFFFFFFull ^ mask);
        }
        __syncthreads();
    }
    block_add<PART_BLOCK>(&a.stats[2 * (t <= a.stat_cap ? t - 1 : a.stat_cap) + 1], kills);
}

static size_t ckill_smem(int r, uint32_t nbins, uint32_t enb) {
    return sizeof(ull) * (size_t)(r - 1) * CKCH + (sizeof(ull) + 2 * sizeof(uint32_t)) * nbins +
           sizeof(uint32_t) * (enb + 1);
}

// ---- apply: the round's decrements bin-major, DCH entries per work item (a counter hands
// them out in bin order, so the blocks in flight share about one bin).  COMPACT: a decrement
// first looks up its vertex's record; a vertex without a slot (it left before the last
// compaction) is skipped.  A returning 64-bit atomic per decrement; the one that sees
// count == k makes the crossing.
template <int R, bool COMPACT>
__global__ void __launch_bounds__(CB_BLOCK, 6) capply_kernel(CArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t fen;
    __shared__ ull item[2];  // double-buffered: no barrier needed before the next claim
    const uint32_t nb = a.nbins;
    if (a.rc && *(volatile uint32_t *)&a.rc->stop) return;  // uniform: the loop stopped before this round
    const uint32_t t = a.rc ? *(volatile uint32_t *)&a.rc->t : a.t;
    // (a select, not a.fec[t & 1]: a dynamic index into a kernel parameter copies the whole
    // parameter struct to local memory -- 248 bytes of stack, +6 ms of apply at C5)
    const FeView f = fe_view<FE_CAP_A>(smem_raw, a.enb, &fen, a.rc ? ((t & 1) ? a.fec[1] : a.fec[0]) : a.fecnt);
    uint32_t *pre = (uint32_t *)(f.offs + a.enb);  // [nb + 1] items before bin b
    if (threadIdx.x == 0) fen = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += CB_BLOCK) pre[b] = (uint32_t)((ld_cg_u64(a.cursor + b) + CDCH - 1) / CDCH);
    block_excl_scan(pre, nb);
    const uint32_t nitems = pre[nb];
    const ull mask = (1ull << BIN_SHIFT) - 1;
    const uint32_t k = a.k;
    ull crossed = 0;
    for (int ib = 0;; ib ^= 1) {
        if (threadIdx.x == 0) item[ib] = atomicAdd(a.work, 1ull);
        __syncthreads();
        const ull c = item[ib];
        if (c >= nitems) break;
        uint32_t lo = 0, hi = nb;  // bin b with pre[b] <= c < pre[b+1]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= c) lo = mid; else hi = mid;
        }
        const uint32_t b = lo, j = (uint32_t)c - pre[b];
        if (threadIdx.x == 0 && b + 1 < nb) {
            // slice j of the next bin's slots (and records) into L2
            const uint32_t nj = pre[b + 1] - pre[b];
            const uint64_t sb = (COMPACT ? ld_cg_u64(a.slots + b + 1) : bin_size(a.n, b + 1)) * sizeof(ull);
            const uint64_t ss = ((sb + nj - 1) / nj + 15) & ~15ull, so = (uint64_t)j * ss;
            if (so < sb)
                prefetch_l2((const char *)(a.X + ((uint64_t)(b + 1) << BIN_SHIFT)) + so,
                            (uint32_t)min((ull)ss, (ull)((sb - so + 15) & ~15ull)));
            if (COMPACT) {
                const uint64_t rb = bin_groups(a.n, b + 1) * sizeof(CRec);
                const uint64_t rs = ((rb + nj - 1) / nj + 15) & ~15ull, ro = (uint64_t)j * rs;
                if (ro < rb)
                    prefetch_l2((const char *)(a.recs + ((uint64_t)(b + 1) << (BIN_SHIFT - 6))) + ro,
                                (uint32_t)min((ull)rs, (ull)((rb - ro + 15) & ~15ull)));
            }
        }
#if PEEL_CAPPLY_PF
        if (threadIdx.x == 32) {  // the entries of the item one wave ahead into L2
            const ull c2 = c + gridDim.x;
            if (c2 < nitems) {
                uint32_t lo2 = 0, hi2 = nb;
                while (hi2 - lo2 > 1) {
                    const uint32_t mid = (lo2 + hi2) >> 1;
                    if (pre[mid] <= c2) lo2 = mid; else hi2 = mid;
                }
                const uint32_t j2 = (uint32_t)c2 - pre[lo2];
                const ull cnt2 = ld_cg_u64(a.cursor + lo2);
                const ull n2 = min((ull)CDCH, cnt2 - (ull)j2 * CDCH);
                const char *p2 = (const char *)(a.entries + a.base[lo2] + (ull)j2 * CDCH);
                const uintptr_t q0 = (uintptr_t)p2 & ~(uintptr_t)15, q1 = ((uintptr_t)p2 + n2 * 8 + 15) & ~(uintptr_t)15;
                prefetch_l2((const void *)q0, (uint32_t)(q1 - q0));
            }
        }
#endif
        const ull cnt = ld_cg_u64(a.cursor + b);
        const ull *ent = a.entries + a.base[b] + (ull)j * CDCH;
        const uint32_t nin = (uint32_t)min((ull)CDCH, cnt - (ull)j * CDCH);
        ull *st = a.X + ((uint64_t)b << BIN_SHIFT);
        const CRec *rb = a.recs + ((uint64_t)b << (BIN_SHIFT - 6));
        // all DU entries of a thread: loads, record lookups and returning atomics issued before
        // any result is used
        constexpr int DU = CDCH / CB_BLOCK;
        ull x[DU], old[DU];
        #pragma unroll
        for (int r = 0; r < DU; r++) {
            const uint32_t i = threadIdx.x + r * CB_BLOCK;
            x[r] = i < nin ? __ldcs(ent + i) : 0ull;
        }
        int64_t slot[DU];
        #pragma unroll
        for (int r = 0; r < DU; r++) {
            const uint32_t i = threadIdx.x + r * CB_BLOCK;
            slot[r] = -1;
            if (i >= nin) continue;
            if (COMPACT) {
                const uint4 rc = __ldcg(reinterpret_cast<const uint4 *>(rb + ((x[r] & mask) >> 6)));
                const ull m = ((ull)rc.y << 32) | rc.x;
                const uint32_t bit = (uint32_t)x[r] & 63u;
                if ((m >> bit) & 1ull) slot[r] = (int64_t)rc.z + __popcll(m & ((1ull << bit) - 1ull));
            } else {
                slot[r] = (int64_t)(((uint64_t)b << BIN_SHIFT) + (x[r] & mask));
            }
        }
        #pragma unroll
        for (int r = 0; r < DU; r++) {
            old[r] = 0;
            if (slot[r] >= 0) old[r] = atomicAdd(a.X + slot[r], 0ull - ((x[r] & ~0xFFFFFFFFull) + 1ull));
        }
        (void)st;
        #pragma unroll
        for (int r = 0; r < DU; r++) {
            if (slot[r] >= 0 && count_of(old[r]) == k) {
                crossed++;
                const uint32_t u = (uint32_t)((b << BIN_SHIFT) + (uint32_t)(x[r] & mask));
                if (a.peel_round) a.peel_round[u] = t + 1;
                fe_push<FE_CAP_A>(f, a, make_uint2(u, idsum_of(old[r]) - (uint32_t)(x[r] >> 32)));
            }
        }
        __syncthreads();  // every push of this item landed: one flush decision for the block
        if (fen >= FE_CAP_A / 2) fe_flush<FE_CAP_A>(f, a);
    }
    fe_flush<FE_CAP_A>(f, a);
    block_add<CB_BLOCK>(&a.ctl->nf[t % 3], crossed);
    block_add<CB_BLOCK>(&a.ctl->ne[t % 3], crossed);
}

static size_t capply_smem(uint32_t nbins, uint32_t enb) { return fe_smem(FE_CAP_A, enb) + sizeof(uint32_t) * (nbins + 1); }

// ---- end of the path
// core_mask[v] = count(slot(v)) >= k, 0 without a slot: one record per thread, 64 mask bytes
__global__ void __launch_bounds__(256) cmask_kernel(const CRec *__restrict__ recs, const ull *__restrict__ X, uint64_t n,
                                                    uint32_t k, uint8_t *mask, int vec) {
    const uint64_t ng = (n + 63) >> 6;
    for (uint64_t g = blockIdx.x * 256ull + threadIdx.x; g < ng; g += (uint64_t)gridDim.x * 256) {
        const uint4 r = __ldcs(reinterpret_cast<const uint4 *>(recs + g));
        ull m = ((ull)r.y << 32) | r.x;
        // live = slot and count >= k (a vertex that left since the last compaction keeps its slot)
        ull live = 0;
        uint32_t idx = r.z;
        for (ull mm = m; mm; mm &= mm - 1) {
            const int bit = __ffsll((long long)mm) - 1;
            if ((uint32_t)__ldcs(X + idx) >= k) live |= 1ull << bit;
            idx++;
        }
        m = live;
        const uint64_t v0 = g << 6;
        if (vec && v0 + 64 <= n) {
            uint4 *o = reinterpret_cast<uint4 *>(mask + v0);
            #pragma unroll
            for (int q = 0; q < 4; q++) {
                uint32_t w[4];
                #pragma unroll
                for (int x = 0; x < 4; x++) {
                    const uint32_t bits = (uint32_t)(m >> (16 * q + 4 * x)) & 0xFu;
                    w[x] = (bits & 1u) | ((bits >> 1) & 1u) << 8 | ((bits >> 2) & 1u) << 16 | ((bits >> 3) & 1u) << 24;
                }
                o[q] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        } else {
            for (uint64_t v = v0; v < v0 + 64 && v < n; v++) mask[v] = (uint8_t)((m >> (v - v0)) & 1ull);
        }
    }
}

// core_mask[v] = count(state[v]) >= k (identity slots): 16-byte state loads, 2-byte stores
__global__ void __launch_bounds__(256) cmask_ident_kernel(const ull *__restrict__ state, uint64_t n, uint32_t k,
                                                          uint8_t *mask, int vec) {
    const uint64_t np = vec ? n / 2 : 0;
    for (uint64_t p = blockIdx.x * 256ull + threadIdx.x; p < np; p += (uint64_t)gridDim.x * 256) {
        const uint4 x = __ldcs(reinterpret_cast<const uint4 *>(state) + p);
        reinterpret_cast<uint16_t *>(mask)[p] = (uint16_t)((x.x >= k) | (x.z >= k) << 8);
    }
    for (uint64_t v = np * 2 + blockIdx.x * 256ull + threadIdx.x; v < n; v += (uint64_t)gridDim.x * 256)
        mask[v] = (uint32_t)state[v] >= k ? 1 : 0;
}

// the full state array back from the slots for the persistent tail: a vertex with a slot gets
// its state; any other vertex left before the last compaction (count 0, or 1 in F_t) and gets
// count k - 1, id sum 0 -- a decrement never reaches it with count k (a dead vertex gets
// none, a frontier vertex at most one), and its entry carries its edge
__global__ void __launch_bounds__(256) cdecompact_kernel(const CRec *__restrict__ recs, const ull *__restrict__ X,
                                                         uint64_t n, uint32_t k, ull *state) {
    for (uint64_t v = blockIdx.x * 256ull + threadIdx.x; v < n; v += (uint64_t)gridDim.x * 256) {
        const uint4 r = __ldg(reinterpret_cast<const uint4 *>(recs + (v >> 6)));
        const ull m = ((ull)r.y << 32) | r.x;
        const uint32_t bit = (uint32_t)v & 63u;
        state[v] = ((m >> bit) & 1ull) ? __ldcs(X + r.z + __popcll(m & ((1ull << bit) - 1ull))) : (ull)(k - 1);
    }
}

// F_t from the edge-bin regions into one list (the persistent kernel's input)
__global__ void __launch_bounds__(256) cgather_kernel(const uint2 *__restrict__ fe, uint64_t stride,
                                                      const ull *__restrict__ fecur, uint32_t enb, uint2 *out) {
    extern __shared__ ull gpre[];  // [enb + 1]
    if (threadIdx.x == 0) {
        ull acc = 0;
        for (uint32_t j = 0; j < enb; j++) { gpre[j] = acc; acc += fecur[j]; }
        gpre[enb] = acc;
    }
    __syncthreads();
    const ull tot = gpre[enb];
    for (ull i = blockIdx.x * 256ull + threadIdx.x; i < tot; i += (ull)gridDim.x * 256) {
        uint32_t lo = 0, hi = enb;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (gpre[mid] <= i) lo = mid; else hi = mid;
        }
        out[i] = fe[(ull)lo * stride + (i - gpre[lo])];
    }
}

// the decision before round t (see RoundCtl); one block
__global__ void __launch_bounds__(256) cround_ctl_kernel(Ctl *ctl, RoundCtl *rc, RoundRule rule, ull *cursor,
                                                         uint32_t nbins, ull *fec0, ull *fec1, uint32_t enb, ull *work) {
    __shared__ uint32_t go, tt;
    if (threadIdx.x == 0) {
        go = 0;
        if (!rc->stop) {
            if (rc->ran) { rc->t++; rc->ran = 0; }
            const uint32_t t = rc->t;
            const ull nF = ld_cg_u64(&ctl->nf[(t - 1) % 3]), nE = ld_cg_u64(&ctl->ne[(t - 1) % 3]);
            if (t > 1 && rc->live_t != t) { rc->live -= nF; rc->live_t = t; }  // F_t left L in round t-1
            const double live = (double)rc->live, slots = (double)rc->nslots, n = (double)rule.n;
            if (nF == 0) rc->stop = RC_DONE;
            else if ((double)nE < rule.frac * n && live >= rule.tail * n && slots >= rule.tratio * (double)nE)
                rc->stop = RC_TAIL;
            else if (rule.compaction && live <= (rc->nslots == rule.n ? rule.at1 : rule.at) * slots &&
                     8.0 * (slots - live) >= 0.5 * n)
                rc->stop = RC_COMPACT;
            else { go = 1; rc->ran = 1; }
            tt = t;
        }
    }
    __syncthreads();
    if (!go) return;
    ull *fn = (tt & 1) ? fec1 : fec0;
    for (uint32_t i = threadIdx.x; i < nbins; i += 256) cursor[i] = 0ull;
    for (uint32_t i = threadIdx.x; i < enb; i += 256) fn[i] = 0ull;
    if (threadIdx.x == 0) *work = 0ull;
}

// rounds, and the timer that closes the last round (profiling), once the frontier is empty
__global__ void ctail_kernel(Ctl *ctl, ull *rtime, uint32_t T, uint32_t stat_cap) {
    ctl->rounds = T;
    if (T + 1 <= stat_cap) rtime[T] = globaltimer();
}

// ---- host driver ---------------------------------------------------------------------------
static bool compact_on() {
    const char *e = getenv("PEEL_COMPACT");  // read per call: tests and A/B runs toggle it
    return !(e && atoi(e) == 0);
}

// A small frontier with a large live set (above threshold) is cheaper on the persistent
// kernel after one write-back of the full state (8 B per vertex, once): a compacted round
// streams 8 B per SLOT whatever the frontier, the persistent kernel pays per frontier entry
// (a few random 64 B DRAM granules).  Hand over when the live set is >= PEEL_COMPACT_TAIL n
// (default 0.11) and there are >= PEEL_COMPACT_TAIL_RATIO (default 64) slots per entry.
// Measured: C4a 9.70 ms compacted to the end against 7.11 handed over; C3 13.39 against 14.95
// when the live-set rule alone handed its rounds over at the first 5% frontier.
static double ctail_live_frac() {
    const char *e = getenv("PEEL_COMPACT_TAIL");
    return e ? atof(e) : 0.11;
}
static double ctail_ratio() {
    const char *e = getenv("PEEL_COMPACT_TAIL_RATIO");
    return e ? atof(e) : 64.0;
}

// a per-device side stream and two events for work that overlaps the round kernels
struct SideStream {
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
};
static SideStream &side_stream() {
    // per host thread and device: concurrent calls from several threads (peel_sweep's batch
    // workers) must not share the side stream's events
    static thread_local std::map<int, SideStream> per;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); dev = 0; }
    SideStream &sd = per[dev];
    if (!sd.s2) {
        if (cudaStreamCreateWithFlags(&sd.s2, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&sd.ev[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sd.ev[1], cudaEventDisableTiming) != cudaSuccess) {
            set_cuda_error(cudaGetLastError(), "side stream");
            sd.s2 = nullptr;
        }
    }
    return sd;
}

static double compact_at() {
    const char *e = getenv("PEEL_COMPACT_AT");  // live / slots ratio that triggers (A/B; 0: never)
    return e ? atof(e) : 0.5;
}
static double compact_at1() {
    const char *e = getenv("PEEL_COMPACT_AT1");  // the first compaction (identity slots)
    return e ? atof(e) : compact_at();
}
static int rounds_per_sync() {
    const char *e = getenv("PEEL_ROUNDS_PER_SYNC");
    const int k = e ? atoi(e) : 4;
    return k < 1 ? 1 : (k > 64 ? 64 : k);
}

// compaction rule (cround_ctl_kernel): compact when the live set has halved since the slots
// were laid out (PEEL_COMPACT_AT) and the bytes a round would stop prefetching (8 per dropped
// slot) pay for the records pass (n / 2 bytes)

template <int R>
static peel_status run_compact(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t k, uint8_t *core_mask,
                               uint32_t *rounds, uint64_t *survivors, uint64_t *killed, uint32_t cap,
                               uint32_t *peel_round, char *ws, const Layout &L, cudaStream_t s,
                               const EdgeStream *es, PeelArgs &a, bool *fallback) {
    *fallback = false;
    Ctl *ctl = (Ctl *)(ws + L.ctl);
    ull *cursor = (ull *)(ws + L.bin_cursor), *bbase = (ull *)(ws + L.bin_base), *bcap = (ull *)(ws + L.bin_cap);
    ull *entries = (ull *)(ws + L.entries);
    const uint32_t nbins = (uint32_t)L.nbins, enb = (uint32_t)L.cl.enb;
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
        bin_partition_kernel<R><<<num_sms() * pblocks, PART_BLOCK, smem, s>>>(edges, n, m, nbins, cursor, bbase, bcap,
                                                                               entries, &ctl->err, &ctl->binovf, 0ull, n, 0ull);
    } else if (m) {  // chunk by chunk, each after its copy
        for (size_t i = 0; i < es->done.size(); i++) {
            const uint64_t e0 = i * es->chunk, e1 = std::min(m, e0 + es->chunk);
            PEEL_CUDA(cudaStreamWaitEvent(s, es->done[i], 0));
            ProfScope ps("bin_partition", s);
            bin_partition_kernel<R><<<num_sms() * pblocks, PART_BLOCK, smem, s>>>(edges, n, e1, nbins, cursor, bbase,
                                                                                   bcap, entries, &ctl->err,
                                                                                   &ctl->binovf, 0ull, n, e0);
        }
    }
    PEEL_CUDA(cudaGetLastError());
    Ctl h;
    PEEL_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    PEEL_CUDA(cudaStreamSynchronize(s));
    if (h.err) return finish_kcore(n, cap, rounds, survivors, killed, ws, L, a, s);  // EINVAL
    if (h.binovf) {  // adversarial degree skew: the direct build of the uncompacted path
        *fallback = true;
        return PEEL_OK;
    }
    const CompactLayout &CL = L.cl;
    ull *slots[2] = {(ull *)(ws + CL.live0), (ull *)(ws + CL.live1)};
    ull *fecnt[2] = {(ull *)(ws + CL.fecnt0), (ull *)(ws + CL.fecnt1)};
    ull *CB[2] = {(ull *)(ws + L.F0), (ull *)(ws + L.F1)};
    ull *state = (ull *)(ws + L.state);
    CArgs c;
    memset(&c, 0, sizeof c);
    c.edges = edges; c.n = n; c.m = m; c.k = k; c.t = 0;
    c.nbins = nbins; c.enb = enb;
    c.recs = (CRec *)(ws + CL.recs);
    c.fe = (uint2 *)(ws + CL.fe);
    c.fe_stride = CL.fe_stride;
    c.ctl = ctl; c.stats = a.stats; c.stat_cap = a.stat_cap; c.peel_round = peel_round;
    c.cursor = cursor; c.base = bbase; c.entries = entries;
    c.work = &ctl->work;
    c.X = state;  // identity slots until the first compaction
    // build: the full states, F_1 into fecnt[0]
    PEEL_CUDA(cudaMemsetAsync(fecnt[0], 0, sizeof(ull) * enb, s));
    c.fecnt = fecnt[0];
    c.live_total = &ctl->nlive[0];
    {
        const size_t bs = fe_smem(FE_CAP_B, enb);
        PEEL_CUDA(raise_smem((const void *)cbuild_kernel<R>, bs));
        int per_sm = 0;
        PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cbuild_kernel<R>, CB_BLOCK, bs));
        if (per_sm < 1) per_sm = 1;
        void *bargs[] = {&c};
        ProfScope ps("bin_accumulate", s);
        PEEL_CUDA(cudaLaunchCooperativeKernel((void *)cbuild_kernel<R>, num_sms() * per_sm, CB_BLOCK, bargs, bs, s));
    }
    // rounds
    BinRound br;
    memset(&br, 0, sizeof br);
    br.nbins = nbins;
    br.cursor = cursor;
    br.base = bbase;
    br.entries = entries;
    br.work = &ctl->work;
    const size_t ksmem = ckill_smem(R, nbins, enb);
    PEEL_CUDA(raise_smem((const void *)ckill_kernel<R>, ksmem));
    PEEL_CUDA(cudaFuncSetAttribute(ckill_kernel<R>, cudaFuncAttributePreferredSharedMemoryCarveout, 72));
    int kb = 0;
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&kb, ckill_kernel<R>, PART_BLOCK, ksmem));
    kb = kb < 1 ? 1 : kb;
    const size_t asmem = capply_smem(nbins, enb);
    int ab[2] = {0, 0};
    PEEL_CUDA(raise_smem((const void *)capply_kernel<R, false>, asmem));
    PEEL_CUDA(raise_smem((const void *)capply_kernel<R, true>, asmem));
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ab[0], capply_kernel<R, false>, CB_BLOCK, asmem));
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ab[1], capply_kernel<R, true>, CB_BLOCK, asmem));
    int cb = 0;
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cb, ccompact_kernel<true>, CB_BLOCK, 0));
    cb = cb < 1 ? 1 : cb;
    SideStream &sd = side_stream();
    if (!sd.s2) return PEEL_ECUDA;
    const double frac = bin_round_frac(n), tail = ctail_live_frac(), tratio = ctail_ratio();
    const bool compaction = compact_on();
    bool compacted = false;
    int cur = 0;             // compacted: the slots live in CB[cur], their counts per bin in slots[cur]
    PEEL_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    PEEL_CUDA(cudaStreamSynchronize(s));
    uint64_t live = h.nlive[0];
    uint64_t nslots = n;     // slots laid out (identity: every vertex)
    // The rounds run as a device-side loop: cround_ctl_kernel decides before each round (done /
    // tail hand-over / compaction due / run) and zeroes its counters; the host launches
    // PEEL_ROUNDS_PER_SYNC rounds (default 4) at a time and syncs once per batch -- rounds
    // after a stop exit at once -- and does only the work the device cannot: the compaction
    // (a buffer swap) and the hand-over.
    RoundCtl *rc = (RoundCtl *)(ws + CL.rc);
    RoundCtl hrc;
    memset(&hrc, 0, sizeof hrc);
    hrc.t = 1;
    hrc.live_t = 1;  // round 1's F_1 left L in the build: live is already after it
    hrc.live = live;
    hrc.nslots = nslots;
    PEEL_CUDA(cudaMemcpyAsync(rc, &hrc, sizeof hrc, cudaMemcpyHostToDevice, s));
    c.rc = rc;
    c.fec[0] = fecnt[0];
    c.fec[1] = fecnt[1];
    const RoundRule rule = {n, frac, tail, tratio, compact_at(), compact_at1(), compaction ? 1 : 0};
    const int K = rounds_per_sync();
    bool comp_pending = false;
    uint32_t t = 1;
    for (;;) {
        for (int i = 0; i < K; i++) {
            cround_ctl_kernel<<<1, 256, 0, s>>>(ctl, rc, rule, cursor, nbins, fecnt[0], fecnt[1], enb, &ctl->work);
            {
                ProfScope ps("round_kill_partition", s);
                ckill_kernel<R><<<num_sms() * kb, PART_BLOCK, ksmem, s>>>(a, br, c);
            }
            if (comp_pending) {
                PEEL_CUDA(cudaStreamWaitEvent(s, sd.ev[1], 0));
                comp_pending = false;
            }
            {
                ProfScope ps("round_apply", s);
                if (compacted) capply_kernel<R, true><<<num_sms() * (ab[1] < 1 ? 1 : ab[1]), CB_BLOCK, asmem, s>>>(c);
                else capply_kernel<R, false><<<num_sms() * (ab[0] < 1 ? 1 : ab[0]), CB_BLOCK, asmem, s>>>(c);
            }
        }
        PEEL_CUDA(cudaGetLastError());
        PEEL_CUDA(cudaMemcpyAsync(&hrc, rc, sizeof hrc, cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
        PEEL_CUDA(cudaStreamSynchronize(s));
        t = hrc.t;
        if (hrc.stop == RC_RUN) continue;
        if (hrc.stop == RC_DONE) break;
        if (hrc.stop == RC_TAIL) {
            // the persistent kernel takes the remaining rounds from round t
            const ull nE = h.ne[(t - 1) % 3];
            if (compacted) {
                ProfScope ps("compact_writeback", s);
                cdecompact_kernel<<<grid_for(n), 256, 0, s>>>(c.recs, c.X, n, k, state);
            }
            uint2 *Ft = (uint2 *)a.F[(t - 1) & 1];
            {
                ProfScope ps("compact_gather", s);
                cgather_kernel<<<grid_for(nE ? nE : 1), 256, sizeof(ull) * (enb + 1), s>>>(c.fe, c.fe_stride,
                                                                                            fecnt[(t - 1) & 1], enb, Ft);
            }
            a.state = state;
            a.t0 = t;
            a.f1_ready = 1;
            int per_sm = 0;
            PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peel_packed_kernel<R>, PEEL_BLOCK, 0));
            if (per_sm < 1) per_sm = 1;
            void *args[] = {&a};
            {
                ProfScope ps("peel_rounds_packed", s);
                PEEL_CUDA(cudaLaunchCooperativeKernel((void *)peel_packed_kernel<R>, num_sms() * per_sm, PEEL_BLOCK,
                                                      args, 0, s));
            }
            return finish_kcore(n, cap, rounds, survivors, killed, ws, L, a, s);
        }
        // RC_COMPACT: lay the live states out densely -- CB[nxt], slot counts slots[nxt], new
        // records -- on the side stream: round t's kill does not touch the slots and runs
        // concurrently; its apply waits for the compaction
        const int nxt = compacted ? cur ^ 1 : 0;
        PEEL_CUDA(cudaEventRecord(sd.ev[0], s));
        PEEL_CUDA(cudaStreamWaitEvent(sd.s2, sd.ev[0], 0));
        PEEL_CUDA(cudaMemsetAsync(slots[nxt], 0, sizeof(ull) * nbins, sd.s2));
        PEEL_CUDA(cudaMemsetAsync(&ctl->cwork, 0, sizeof(ull), sd.s2));
        CArgs cc = c;
        cc.Y = CB[nxt];
        cc.alloc = slots[nxt];
        cc.work = &ctl->cwork;
        {
            ProfScope ps("compact_slots", sd.s2);
            const char *cre = getenv("PEEL_CREG");
            if (!(cre && atoi(cre) == 0)) {
                if (compacted) ccompact_reg_kernel<false><<<num_sms() * cb, CB_BLOCK, 0, sd.s2>>>(cc);
                else ccompact_reg_kernel<true><<<num_sms() * cb, CB_BLOCK, 0, sd.s2>>>(cc);
            } else {
                if (compacted) ccompact_kernel<false><<<num_sms() * cb, CB_BLOCK, 0, sd.s2>>>(cc);
                else ccompact_kernel<true><<<num_sms() * cb, CB_BLOCK, 0, sd.s2>>>(cc);
            }
        }
        PEEL_CUDA(cudaEventRecord(sd.ev[1], sd.s2));
        comp_pending = true;
        compacted = true;
        cur = nxt;
        c.X = CB[cur];
        c.slots = slots[cur];
        hrc.nslots = hrc.live;
        hrc.stop = RC_RUN;
        PEEL_CUDA(cudaMemcpyAsync(rc, &hrc, sizeof hrc, cudaMemcpyHostToDevice, s));
    }
    {
        ProfScope ps("compact_core_mask", s);
        ctail_kernel<<<1, 1, 0, s>>>(ctl, a.rtime, t - 1, a.stat_cap);
        if (compacted) cmask_kernel<<<grid_for((n + 63) / 64), 256, 0, s>>>(c.recs, c.X, n, k, core_mask, a.mask_vec);
        else cmask_ident_kernel<<<grid_for(n / 2 + 1), 256, 0, s>>>(state, n, k, core_mask, a.mask_vec);
    }
    PEEL_CUDA(cudaGetLastError());
    return finish_kcore(n, cap, rounds, survivors, killed, ws, L, a, s);
}
