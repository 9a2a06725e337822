// dist.cu -- e2: one peeling instance partitioned by vertex range over P GPUs
// (BASELINE.json configs[4] "vertex-partitioned single instance").
//
// Rank p owns vertices [p n / P, (p+1) n / P): their packed state (Σ edge ids << 32 | count),
// frontier entries and core-mask slice.  The edge list is replicated read-only, and each
// rank keeps its own m-bit alive bitmap, meaningful for edges touching its vertices.
// A round (k = 2, the round-synchronous schedule of P:48-50):
//   kill    for each local frontier entry (v, e): test-and-clear alive_p[e]; the winner
//           decrements its own endpoints of e (crossing 2 -> 1 appends (u, Σ - e) to the
//           local F_{t+1}) and queues e for every OTHER rank owning an endpoint of e;
//   exchange  one all-to-all of the queued edge ids (NCCL grouped send/recv; or device
//           copies between virtual shards of one GPU);
//   receive each received e: test-and-clear alive_q[e]; the winner decrements its own
//           endpoints of e.  Every (e, rank) pair is applied exactly once -- by that rank's
//           test-and-clear -- even when several ranks kill e in the same round;
//   stats   allreduce of (|F_{t+1}|, edges killed) -- an edge's kill is counted by the
//           owner of its smallest endpoint -- the termination test.
// Bit-exact with the single-GPU peel by construction: every vertex's count sees exactly
// the decrements of its killed edges, and F_{t+1} is the set of k -> k-1 crossings.
#include <nccl.h>
#include <stdlib.h>
#include <stddef.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <vector>

#include "common.cuh"
#include "shard.h"
#include "comm.h"

namespace peel {

static constexpr int DB = 256;            // block size
static constexpr int DQ = 2 * DB;         // block-queue capacity

struct DCtl {
    ull nf[2];      // |F_t| local, double-buffered by round parity
    ull ne[2];      // frontier entry counts
    ull kills;      // edges killed this round, counted at the owner of the smallest endpoint
    ull nsend[8];   // per-destination queue lengths this round
    ull fail;       // this rank failed locally (host status != OK): the error word of the
                    // count exchange, right after nsend (one 9-word allgather per round)
    uint32_t err;
    uint32_t pad;
};
static_assert(offsetof(DCtl, fail) == offsetof(DCtl, nsend) + 8 * sizeof(ull), "count row = nsend[8], fail");

// the per-round reset clears kills and nsend[8] with one memset
static_assert(offsetof(DCtl, nsend) == offsetof(DCtl, kills) + sizeof(ull), "per-round counters contiguous");

static inline size_t dal(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline uint64_t shard_lo(uint64_t n, int P, int q) { return (uint64_t)q * n / (uint64_t)P; }

// owner of u: the number of shard boundaries lo[1 .. P-1] at or below u (P <= 8 compares)
__device__ __forceinline__ int owner_fast(uint32_t u, const uint32_t (&lo)[8], int P) {
    int q = 0;
    #pragma unroll
    for (int i = 1; i < 8; i++) q += (i < P) && u >= lo[i];
    return q;
}

__device__ __forceinline__ int owner_of(uint32_t u, uint64_t n, int P) {
    int q = (int)(((uint64_t)u * (uint64_t)P) / n);
    if (q >= P) q = P - 1;
    while (q > 0 && (uint64_t)u < shard_lo(n, P, q)) q--;
    while (q + 1 < P && (uint64_t)u >= shard_lo(n, P, q + 1)) q++;
    return q;
}

struct DShard {
    int q;                 // shard index (= rank for NCCL)
    uint64_t v0, v1;       // owned vertices
    ull *state;            // [v1 - v0]
    uint32_t *alive;       // [m/32]
    uint2 *F[2];           // frontier entries (global v, e), cap v1 - v0
    uint32_t *send;        // P segments of cap (v1 - v0) each
    uint32_t *recv;        // cap n
    DCtl *ctl;
    bool binned;           // the shard was built binned: its bins serve the binned rounds
    char *bins;            // shard_build scratch
};

struct DLayout {
    size_t ctl, scratch, state, alive, F0, F1, send, recv, bins, bins_bytes, total;
};

static DLayout dlayout(uint64_t n, uint64_t m, uint32_t r, int P, uint64_t nloc) {
    DLayout L;
    size_t o = 0;
    L.ctl = o; o += dal(sizeof(DCtl));
    L.scratch = o; o += dal(sizeof(ull) * (8 + 9 * 8 + 5 * 8));  // collective staging: sums, P count rows, pack words
    L.state = o; o += dal(sizeof(ull) * nloc);
    L.alive = o; o += dal(sizeof(uint32_t) * ((m + 31) / 32));
    L.F0 = o; o += dal(sizeof(uint2) * nloc);
    L.F1 = o; o += dal(sizeof(uint2) * nloc);
    L.send = o; o += dal(sizeof(uint32_t) * nloc * P);
    L.recv = o; o += dal(sizeof(uint32_t) * n);
    L.bins_bytes = shard_build_bytes(n, m, r, nloc);  // 0: the shard builds directly
    L.bins = o; o += dal(L.bins_bytes);
    L.total = o;
    return L;
}

typedef BlockQueueT<uint2, DQ, DB> DEntQ;
typedef BlockQueueT<uint32_t, DQ, DB> DIdQ;

// flush the P per-destination send queues with two block barriers in all (bq_flush per
// queue would take two each): thread 0 reserves every non-empty queue's output range, then
// the block copies them out.  Every thread of the block must call it.
__device__ __forceinline__ void flush_sends(DIdQ *qs, int slot, uint32_t P, uint32_t *send, uint64_t nloc,
                                            ull *nsend) {
    __syncthreads();
    if (threadIdx.x == 0)
        for (uint32_t d = 0; d < P; d++) {
            const uint32_t c = min(qs[d].n[slot], (uint32_t)DQ);
            qs[d].cnt = c;
            qs[d].base = c ? atomicAdd(nsend + d, (ull)c) : 0ull;
            qs[d].n[slot] = 0;
        }
    __syncthreads();
    for (uint32_t d = 0; d < P; d++) {
        const uint32_t c = qs[d].cnt;
        const ull b = qs[d].base;
        for (uint32_t i = threadIdx.x; i < c; i += DB) send[(uint64_t)d * nloc + b + i] = qs[d].buf[slot][i];
    }
}

template <int R>
__device__ __forceinline__ bool dload_edge(const uint32_t *__restrict__ edges, uint64_t e, uint64_t n,
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

// build: every rank scans all edges, accumulates its own endpoints
template <int R>
__global__ void __launch_bounds__(DB) dist_build_kernel(const uint32_t *__restrict__ edges, uint64_t n, uint64_t m,
                                                        uint64_t v0, uint64_t v1, ull *state, DCtl *ctl) {
    for (uint64_t e = blockIdx.x * (uint64_t)DB + threadIdx.x; e < m; e += (uint64_t)gridDim.x * DB) {
        uint32_t u[R];
        if (!dload_edge<R>(edges, e, n, u)) {
            atomicOr(&ctl->err, 1u);
            continue;
        }
        const ull inc = (e << 32) + 1ull;
        #pragma unroll
        for (int j = 0; j < R; j++)
            if (u[j] >= v0 && u[j] < v1) atomicAdd(state + (u[j] - v0), inc);
    }
}

// round 1: F_1 over owned vertices
__global__ void __launch_bounds__(DB) dist_scan_kernel(const ull *__restrict__ state, uint64_t v0, uint64_t nloc,
                                                       uint32_t k, uint2 *F, DCtl *ctl) {
    __shared__ DEntQ q;
    bq_init(q);
    __syncthreads();
    ull removed = 0;
    int slot = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * DB; base < nloc; base += (uint64_t)gridDim.x * DB) {
        const uint64_t i = base + threadIdx.x;
        if (i < nloc) {
            const ull w = state[i];
            if ((uint32_t)w < k) {
                removed++;
                if ((uint32_t)w == 1u) bq_push(q, slot, make_uint2((uint32_t)(v0 + i), (uint32_t)(w >> 32)), F, &ctl->ne[1]);
            }
        }
        bq_flush(q, slot, F, &ctl->ne[1]);
        slot ^= 1;
    }
    block_add<DB>(&ctl->nf[1], removed);
}

// decrement owned endpoint u of killed edge e; crossing count 2 -> 1 joins F_{t+1}
__device__ __forceinline__ void dist_decrement(ull *state, uint64_t v0, uint32_t u, uint32_t e, uint32_t k,
                                               DEntQ &q, int slot, uint2 *Fn, ull *cn, ull &crossed) {
    const ull old = atomicAdd(state + (u - v0), 0ull - (((ull)e << 32) + 1ull));
    if ((uint32_t)old == k) {
        crossed++;
        bq_push(q, slot, make_uint2(u, (uint32_t)(old >> 32) - e), Fn, cn);
    }
}

struct DKArgs {
    const uint32_t *edges;
    uint64_t n, m;
    uint32_t lo[8];  // shard boundaries lo[q] = shard_lo(n, P, q) for q < P (lo[0] = 0): owner
                     // lookups by comparison, not a 64-bit division per endpoint
    int edges_vec;  // edges is 16-byte aligned (vector row loads)
    int P, p;
    uint32_t k;
    uint64_t v0, v1, nloc;
    ull *state;
    uint32_t *alive;
    const uint2 *Fc;
    ull nE;
    uint2 *Fn;
    uint32_t *send;
    DCtl *ctl;
    int par;  // parity of round t+1's counters
};

// kill: local frontier entries
template <int R>
__global__ void __launch_bounds__(DB) dist_kill_kernel(DKArgs a) {
    __shared__ DEntQ q;
    __shared__ DIdQ qs[8];
    bq_init(q);
    for (int d = 0; d < 8; d++) bq_init(qs[d]);
    __syncthreads();
    ull *cn = &a.ctl->ne[a.par];
    ull crossed = 0, kills = 0;
    int slot = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * DB; base < a.nE; base += (uint64_t)gridDim.x * DB) {
        const uint64_t i = base + threadIdx.x;
        if (i < a.nE) {
            const uint2 ent = __ldcg(a.Fc + i);
            const uint32_t e = ent.y, bit = 1u << (e & 31);
            if (atomicAnd(a.alive + (e >> 5), ~bit) & bit) {
                uint32_t u[R];
                uint32_t mn = 0xFFFFFFFFu;
                load_row<R>(a.edges, e, a.m, a.edges_vec, u);
                #pragma unroll
                for (int j = 0; j < R; j++) mn = min(mn, u[j]);
                if (owner_fast(mn, a.lo, a.P) == a.p) kills++;
                uint32_t sent_mask = 0;
                #pragma unroll
                for (int j = 0; j < R; j++) {
                    const int o = owner_fast(u[j], a.lo, a.P);
                    if (o == a.p) {
                        if (u[j] != ent.x) dist_decrement(a.state, a.v0, u[j], e, a.k, q, slot, a.Fn, cn, crossed);
                    } else {
                        sent_mask |= 1u << o;
                    }
                }
                // one push per destination rank; d is warp-uniform, so each coalesced
                // group inside bq_push targets a single queue
                for (int d = 0; d < a.P; d++)
                    if (sent_mask >> d & 1u) bq_push(qs[d], slot, e, a.send + (uint64_t)d * a.nloc, &a.ctl->nsend[d]);
            }
        }
        bq_flush(q, slot, a.Fn, cn);
        flush_sends(qs, slot, a.P, a.send, a.nloc, a.ctl->nsend);
        slot ^= 1;
    }
    block_add<DB>(&a.ctl->nf[a.par], crossed);
    block_add<DB>(&a.ctl->kills, kills);
}

// receive: edge ids killed by other ranks this round
template <int R>
__global__ void __launch_bounds__(DB) dist_recv_kernel(DKArgs a, const uint32_t *__restrict__ recv, ull nrecv) {
    __shared__ DEntQ q;
    bq_init(q);
    __syncthreads();
    ull *cn = &a.ctl->ne[a.par];
    ull crossed = 0, kills = 0;
    int slot = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * DB; base < nrecv; base += (uint64_t)gridDim.x * DB) {
        const uint64_t i = base + threadIdx.x;
        if (i < nrecv) {
            const uint32_t e = __ldcg(recv + i), bit = 1u << (e & 31);
            if (atomicAnd(a.alive + (e >> 5), ~bit) & bit) {
                uint32_t mn = 0xFFFFFFFFu;
                uint32_t u[R];
                load_row<R>(a.edges, e, a.m, a.edges_vec, u);
                #pragma unroll
                for (int j = 0; j < R; j++) mn = min(mn, u[j]);
                if (owner_fast(mn, a.lo, a.P) == a.p) kills++;
                #pragma unroll
                for (int j = 0; j < R; j++)
                    if (u[j] >= a.v0 && u[j] < a.v1) dist_decrement(a.state, a.v0, u[j], e, a.k, q, slot, a.Fn, cn, crossed);
            }
        }
        bq_flush(q, slot, a.Fn, cn);
        slot ^= 1;
    }
    block_add<DB>(&a.ctl->nf[a.par], crossed);
    block_add<DB>(&a.ctl->kills, kills);
}

// ---- binned rounds on a shard (large local frontiers) -------------------------------------
// Same split as the single-GPU binned rounds (kcore.cu): the kill kernel stages the round's
// decrements of OWNED endpoints in the shard's vertex bins (shared-memory counting sort, one
// global atomic per bin per chunk, coalesced runs) instead of applying them as random
// read-modify-writes; shard_apply then applies them bin by bin with L2-resident atomics.
// RECV = false: entries are the local frontier (v, e), remote owners are sent e;
// RECV = true: entries are edge ids received from other shards.
// 3 entries per thread at 5 resident blocks per SM (48 registers): C5 over 8 virtual shards
// 237.4 -> 215.6 ms against 4 at 4 (64 registers); 4 at 5: 222.9, 3 at 4: 221.5, 3 at 6: 227.9
#ifndef PEEL_DKU
#define PEEL_DKU 3
#endif
#ifndef PEEL_DKB_MINB
#define PEEL_DKB_MINB 5
#endif
static constexpr int DKU = PEEL_DKU;           // entries per thread per chunk
static constexpr int DKCH = DB * DKU;          // entries per chunk

static size_t dist_stage_smem(int r, uint32_t nbins) {  // nbins + 8: room for the destinations
    return sizeof(ull) * (size_t)r * DKCH + (sizeof(ull) + 2 * sizeof(uint32_t)) * (nbins + 8);
}

template <int R, bool RECV>
__global__ void __launch_bounds__(DB, PEEL_DKB_MINB) dist_kill_bin_kernel(DKArgs a, const uint32_t *__restrict__ recv, ull nrecv,
                                                            ShardBinsView bv) {
    extern __shared__ unsigned char smem_raw[];
    constexpr int SE = R * DKCH;
    const uint32_t nbins = bv.nbins;
    // the kill's sends are ranked and written with the owned decrements: destination d is
    // "bin" nbins + d of the same counting sort (one scan, one global atomic per destination
    // and chunk, coalesced runs into its send segment) -- round 2; it replaced P block queues
    // (32 KB of static shared memory) and a per-destination push loop per entry
    const uint32_t nbx = RECV ? nbins : nbins + (uint32_t)a.P;  // bins + destinations
    ull *sorted = (ull *)smem_raw;                // [SE] the chunk's decrements and sends, bin-sorted
    ull *gpos = sorted + SE;                      // [nbx]
    uint32_t *hist = (uint32_t *)(gpos + nbx);    // [nbx]
    uint32_t *offs = hist + nbx;                  // [nbx]
    __shared__ uint32_t total;
    const ull nE = RECV ? nrecv : a.nE;
    const ull lmask = (1ull << SHARD_BIN_SHIFT) - 1;
    ull kills = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * DKCH; base < nE; base += (uint64_t)gridDim.x * DKCH) {
        for (uint32_t b = threadIdx.x; b < nbx; b += DB) hist[b] = 0;
        uint2 ent[DKU];
        bool win[DKU];
        #pragma unroll
        for (int j = 0; j < DKU; j++) {
            const uint64_t i = base + (uint64_t)j * DB + threadIdx.x;
            if (RECV) ent[j] = make_uint2(0xFFFFFFFFu, i < nE ? __ldcg(recv + i) : 0u);
            else ent[j] = i < nE ? __ldcg(a.Fc + i) : make_uint2(0u, 0u);
        }
        #pragma unroll
        for (int j = 0; j < DKU; j++) {
            const uint64_t i = base + (uint64_t)j * DB + threadIdx.x;
            win[j] = false;
            if (i < nE) {
                const uint32_t e = ent[j].y, bit = 1u << (e & 31);
                win[j] = (atomicAnd(a.alive + (e >> 5), ~bit) & bit) != 0;
            }
        }
        uint32_t u[DKU][R];
        uint32_t sendm[DKU];
        #pragma unroll
        for (int j = 0; j < DKU; j++) {
            sendm[j] = 0;
            if (!win[j]) continue;
            load_row<R>(a.edges, ent[j].y, a.m, a.edges_vec, u[j]);
            uint32_t mn = 0xFFFFFFFFu;
            #pragma unroll
            for (int r = 0; r < R; r++) {
                mn = min(mn, u[j][r]);
                if (!(u[j][r] >= a.v0 && u[j][r] < a.v1)) sendm[j] |= 1u << owner_fast(u[j][r], a.lo, a.P);
            }
            if (owner_fast(mn, a.lo, a.P) == a.p) kills++;
        }
        __syncthreads();  // hist zeroed
        // owned decrements stay in registers with their rank in the bin (the histogram atomic's
        // return value) until the bin offsets are known (as round_kill_partition_kernel does)
        uint32_t rk[DKU][R];
        #pragma unroll
        for (int j = 0; j < DKU; j++)
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (win[j] && u[j][r] >= a.v0 && u[j][r] < a.v1 && (RECV || u[j][r] != ent[j].x))
                    rk[j][r] = atomicAdd(&hist[(uint32_t)(u[j][r] - a.v0) >> SHARD_BIN_SHIFT], 1u);
        uint32_t rs[DKU][R - 1];  // ranks of the entry's sends, in the order of its destination bits
        if (!RECV) {
            #pragma unroll
            for (int j = 0; j < DKU; j++) {
                uint32_t sm = sendm[j];
                #pragma unroll
                for (int t = 0; t < R - 1; t++)
                    if (sm) {
                        const uint32_t d = __ffs(sm) - 1;
                        sm &= sm - 1;
                        rs[j][t] = atomicAdd(&hist[nbins + d], 1u);
                    }
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t per = (nbx + 31) / 32;
            uint32_t loc = 0;
            for (uint32_t q2 = 0; q2 < per; q2++) {
                uint32_t b = threadIdx.x * per + q2;
                loc += b < nbx ? hist[b] : 0;
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
                if (b < nbx) { offs[b] = run; run += hist[b]; }
            }
            if (threadIdx.x == 31) total = z;
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nbx; b += DB)
            if (hist[b])
                gpos[b] = b < nbins ? atomicAdd(bv.cursor + b, (ull)hist[b])
                                    : (ull)(b - nbins) * a.nloc + atomicAdd(&a.ctl->nsend[b - nbins], (ull)hist[b]);
        #pragma unroll
        for (int j = 0; j < DKU; j++)
            #pragma unroll
            for (int r = 0; r < R; r++)
                if (win[j] && u[j][r] >= a.v0 && u[j][r] < a.v1 && (RECV || u[j][r] != ent[j].x)) {
                    const uint32_t lu = (uint32_t)(u[j][r] - a.v0);
                    sorted[offs[lu >> SHARD_BIN_SHIFT] + rk[j][r]] = ((ull)ent[j].y << 32) | lu;
                }
        if (!RECV) {
            #pragma unroll
            for (int j = 0; j < DKU; j++) {
                uint32_t sm = sendm[j];
                #pragma unroll
                for (int t = 0; t < R - 1; t++)
                    if (sm) {
                        const uint32_t d = __ffs(sm) - 1;
                        sm &= sm - 1;
                        sorted[offs[nbins + d] + rs[j][t]] = ((ull)ent[j].y << 32) | ((nbins + d) << SHARD_BIN_SHIFT);
                    }
            }
        }
        __syncthreads();
        const uint32_t tot = total;
        for (uint32_t i = threadIdx.x; i < tot; i += DB) {
            const ull v = sorted[i];
            const uint32_t b = (uint32_t)v >> SHARD_BIN_SHIFT;
            if (RECV || b < nbins) bv.entries[bv.base[b] + gpos[b] + (i - offs[b])] = v & ~(0xFFFFFFFFull ^ lmask);
            else a.send[gpos[b] + (i - offs[b])] = (uint32_t)(v >> 32);
        }
        __syncthreads();
    }
    block_add<DB>(&a.ctl->kills, kills);
}

__global__ void dist_mask_kernel(const ull *__restrict__ state, uint64_t nloc, uint32_t k, uint8_t *mask) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nloc; i += (uint64_t)gridDim.x * blockDim.x)
        mask[i] = (uint32_t)state[i] >= k ? 1 : 0;
}

// binned-round threshold for a shard of nloc vertices: as kcore.cu's bin_round_frac
static double dist_bin_frac(uint64_t nloc) {
    const char *e = getenv("PEEL_BIN_ROUND_FRAC");
    if (e) {
        const double f = atof(e);
        return f > 0.0 ? f : 2.0;  // 0 disables (no frontier reaches 2 nloc)
    }
    // unlike the single-GPU path, a small local frontier costs the shard random kills, send
    // queues AND a random receive pass: binned rounds pay off from 0.02 nloc once the shard
    // state is >= 0.8 GB (C5 virtual 8 shards 338 -> 311 ms, 4 shards 231 -> 197 ms; C3 at
    // P = 1 19.2 -> 17.6 ms; C3 / C4a over 4 shards of 2.5e7 stay faster at 0.05)
    return 8.0 * (double)nloc >= 8e8 ? 0.02 : 0.05;
}

static unsigned dgrid(uint64_t work) {
    uint64_t b = (work + DB - 1) / DB, cap = (uint64_t)num_sms() * 8;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace peel

using namespace peel;

// per-round bookkeeping of all local shards in one launch each (virtual shards: 8 shards' worth
// of memsets, row copies, packs and 56 exchange copies per round were ~180 small operations,
// whose fixed costs showed as ~17 ms of gaps in C5 over 8 virtual shards)
struct ShardCtls {
    DCtl *c[8];
    ull *z0[8], *z1[8];     // binned shards: the bins' cursors and the edge-sort counters,
    uint32_t n0[8], n1[8];  // zeroed with the round's counters when the shard runs binned
    int n;
};
__global__ void dist_reset_kernel(ShardCtls cs, int nxt, uint32_t binned) {
    const int i = blockIdx.x;
    if (i >= cs.n) return;
    if (threadIdx.x == 0) {
        DCtl *c = cs.c[i];
        c->nf[nxt] = 0;
        c->ne[nxt] = 0;
        c->kills = 0;
        #pragma unroll
        for (int d = 0; d < 8; d++) c->nsend[d] = 0;
    }
    if ((binned >> i) & 1u) {
        for (uint32_t w = threadIdx.x; w < cs.n0[i]; w += blockDim.x) cs.z0[i][w] = 0ull;
        for (uint32_t w = threadIdx.x; w < cs.n1[i]; w += blockDim.x) cs.z1[i][w] = 0ull;
    }
}
// the count rows (nsend[8], fail) of the local shards, shard i at out[9 i]
__global__ void dist_rows_kernel(ShardCtls cs, ull *out) {
    const int i = threadIdx.x / 9, j = threadIdx.x % 9;
    if (i >= cs.n) return;
    out[threadIdx.x] = j < 8 ? cs.c[i]->nsend[j] : cs.c[i]->fail;
}
// virtual exchange: pair p copies cnt[p] ids from src[p] to dst[p] (blockIdx.y = pair)
struct XPairs {
    const uint32_t *src[56];
    uint32_t *dst[56];
    ull cnt[56];
    int n;
};
__global__ void __launch_bounds__(256) dist_xchg_kernel(XPairs x) {
    const int p = blockIdx.y;
    if (p >= x.n) return;
    const ull c = x.cnt[p];
    const uint32_t *src = x.src[p];
    uint32_t *dst = x.dst[p];
    for (ull i = blockIdx.x * 256ull + threadIdx.x; i < c; i += (ull)gridDim.x * 256) dst[i] = __ldcs(src + i);
}

// the end-of-round words of a shard: [0..3] reduced over ranks (|F_{t+1}|, kills, bad-vertex
// bits, failure), [4] local (frontier entries of round t+1, sizes the next kill grid)
__global__ void dist_pack_kernel(ShardCtls cs, int par, ull *out) {
    const int i = threadIdx.x;
    if (i >= cs.n) return;
    const DCtl *ctl = cs.c[i];
    out[5 * i] = ctl->nf[par];
    out[5 * i + 1] = ctl->kills;
    out[5 * i + 2] = ctl->err;
    out[5 * i + 3] = ctl->fail;
    out[5 * i + 4] = ctl->ne[par];
}

static uint64_t max_shard(uint64_t n, int P) {
    uint64_t mx = 0;
    for (int q = 0; q < P; q++) mx = std::max(mx, shard_lo(n, P, q + 1) - shard_lo(n, P, q));
    return mx;
}

extern "C" size_t peel_kcore_dist_workspace_bytes(const peel_comm *c, uint64_t n, uint64_t m, uint32_t r, uint32_t k) {
    if (!c || r < 2 || r > 8 || k > 2 || n > (1ull << 32) || m >= (1ull << 32) || n < (uint64_t)c->P) return 0;
    DLayout L = dlayout(n, m, r, c->P, max_shard(n, c->P));
    return c->virt ? L.total * c->P : L.total;
}

template <int R>
static peel_status run_dist(peel_comm *c, const uint32_t *edges, uint64_t n, uint64_t m, uint32_t k,
                            uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors, uint64_t *killed,
                            uint32_t cap, char *ws, cudaStream_t s) {
    const int P = c->P;
    const uint64_t nl_max = max_shard(n, P);
    const DLayout L = dlayout(n, m, R, P, nl_max);
    // local shards: all P (virtual) or just this rank's
    std::vector<DShard> sh;
    for (int q = 0; q < P; q++) {
        if (!c->virt && q != c->rank) continue;
        char *b = ws + (c->virt ? (size_t)q * L.total : 0);
        DShard d;
        d.q = q;
        d.v0 = shard_lo(n, P, q);
        d.v1 = shard_lo(n, P, q + 1);
        d.ctl = (DCtl *)(b + L.ctl);
        d.state = (ull *)(b + L.state);
        d.alive = (uint32_t *)(b + L.alive);
        d.F[0] = (uint2 *)(b + L.F0);
        d.F[1] = (uint2 *)(b + L.F1);
        d.send = (uint32_t *)(b + L.send);
        d.recv = (uint32_t *)(b + L.recv);
        d.bins = b + L.bins;
        d.binned = false;
        sh.push_back(d);
    }
    // Error protocol (peel.h "Errors"): a rank's first local failure is kept in lst; from then
    // on it launches nothing but still takes part in every collective with its failure word
    // set, and every rank leaves at the next exchange.  Virtual shards have no peers: return.
    const char *ese = getenv("PEEL_ESORT");  // 0: the binned kill takes the frontier unsorted (A/B)
    const bool esort = !(ese && atoi(ese) == 0);
    ShardCtls scs;
    scs.n = (int)sh.size();
    for (int i = 0; i < 8; i++) {
        scs.c[i] = i < scs.n ? sh[i].ctl : nullptr;
        scs.z0[i] = scs.z1[i] = nullptr;
        scs.n0[i] = scs.n1[i] = 0;
        if (i < scs.n && L.bins_bytes && sh[i].v1 > sh[i].v0) {
            const ShardBinsView bv = shard_bins_view(n, m, R, sh[i].v1 - sh[i].v0, sh[i].bins);
            scs.z0[i] = bv.cursor;
            scs.n0[i] = bv.nbins;
            scs.z1[i] = bv.esort;
            scs.n1[i] = bv.esort_words;
        }
    }
    peel_status lst = PEEL_OK;
    auto cu = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess && lst == PEEL_OK) {
            set_cuda_error(e, what);
            lst = PEEL_ECUDA;
        }
        return lst == PEEL_OK;
    };
    auto step = [&](peel_status st2) {
        if (st2 != PEEL_OK && lst == PEEL_OK) lst = st2;
        return lst == PEEL_OK;
    };
    // the binned kill / receive kernels' shared-memory limit, carve-out and resident blocks per
    // SM, set and queried once per (kernel, shared-memory size) in a call, not every round
    std::map<std::pair<bool, size_t>, int> kbc;
    auto kill_blocks = [&](bool recv, size_t sm) -> int {
        auto it = kbc.find({recv, sm});
        if (it != kbc.end()) return it->second;
        const void *kern = recv ? (const void *)dist_kill_bin_kernel<R, true> : (const void *)dist_kill_bin_kernel<R, false>;
        int kb = 0;
        cudaError_t e = raise_smem(kern, sm);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 72);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&kb, kern, DB, sm);
        if (!cu(e, "kill kernel attributes")) return 1;
        kb = kb < 1 ? 1 : kb;
        kbc[{recv, sm}] = kb;
        return kb;
    };
    ull *dsum = (ull *)(ws + L.scratch);  // device staging for the collectives (8 + 8 P words)
    ull one = 1;
    // the failure word of the count exchange (device, read by the gather)
    auto mark_fail = [&]() {
        for (auto &d : sh) cudaMemcpyAsync(&d.ctl->fail, &one, sizeof(ull), cudaMemcpyHostToDevice, s);
    };
    auto leave = [&](bool peer_failed) -> peel_status {
        if (lst != PEEL_OK) return lst;
        return peer_failed ? PEEL_EPEER : PEEL_OK;
    };

    for (auto &d : sh) {
        if (!cu(cudaMemsetAsync(d.ctl, 0, sizeof(DCtl), s), "memset ctl")) break;
        if (!cu(cudaMemsetAsync(d.alive, 0xFF, sizeof(uint32_t) * ((m + 31) / 32), s), "memset alive")) break;
        // large shards: the binned build of kcore.cu restricted to the shard's endpoints
        bool direct = true;
        d.binned = false;
        if (L.bins_bytes && d.v1 - d.v0 > 0) {
            char *b = ws + (c->virt ? (size_t)d.q * L.total : 0);
            // the exchange buffers (send, recv: adjacent) are free during the build
            ShardF1 f1 = {d.F[1], &d.ctl->ne[1], &d.ctl->nf[1], k};  // F_1 from the build's scan
            if (!step(shard_build(R, edges, n, m, d.v0, d.v1, d.state, &d.ctl->err, b + L.bins, s, &direct, b + L.send,
                                  L.bins - L.send, &f1)))
                break;
        }
        d.binned = !direct;  // bins usable by the binned rounds (no overflow)
        if (direct) {  // small shard, or a bin overflowed
            if (!cu(cudaMemsetAsync(d.state, 0, sizeof(ull) * (d.v1 - d.v0), s), "memset state")) break;
            if (m) {
                ProfScope ps("dist_build", s);
                dist_build_kernel<R><<<dgrid(m), DB, 0, s>>>(edges, n, m, d.v0, d.v1, d.state, d.ctl);
            }
        }
        if (direct) {  // a binned build scanned for F_1 itself
            ProfScope ps("dist_scan", s);
            dist_scan_kernel<<<dgrid(d.v1 - d.v0), DB, 0, s>>>(d.state, d.v0, d.v1 - d.v0, k, d.F[1], d.ctl);
        }
    }
    cu(cudaGetLastError(), "build launch");
    if (lst != PEEL_OK && c->virt) return lst;

    // end-of-round words: g[0] = |F_{t+1}|, g[1] = kills, g[2] = bad-vertex bits, g[3] =
    // failed ranks (all global); ne[i] = shard i's frontier entries (local).  ONE stream sync
    // (virtual: the shards' words summed on the host; ranks: one allreduce).
    std::vector<ull> ne(sh.size(), 0), pk(5 * sh.size());
    auto end_round = [&](int par, ull g[4]) -> peel_status {
        if (lst != PEEL_OK) mark_fail();
        dist_pack_kernel<<<1, 32, 0, s>>>(scs, par, dsum + 8);
        const bool nccl = !c->virt && !c->host;
        if (nccl) {  // NCCL: reduce the device words in place, one copy back
            if (!c->nccl) return comm_sync(c, s);  // aborted by the watchdog
            cudaMemcpyAsync(dsum, dsum + 8, sizeof(ull) * 4, cudaMemcpyDeviceToDevice, s);
            ncclResult_t nr = ncclAllReduce(dsum, dsum, 4, ncclUint64, ncclSum, c->nccl, s);
            if (nr != ncclSuccess) { nccl_error(nr); return PEEL_ENCCL; }
            // the watchdog sync, before the copies back: copies to pageable memory block
            // inside the runtime until the stream drains, out of the watchdog's sight
            const peel_status ws = comm_sync(c, s);
            if (ws != PEEL_OK) return lst != PEEL_OK ? lst : ws;
            cudaMemcpyAsync(g, dsum, sizeof(ull) * 4, cudaMemcpyDeviceToHost, s);
        }
        if (cudaMemcpyAsync(pk.data(), dsum + 8, sizeof(ull) * 5 * sh.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            cu(cudaGetLastError(), "end of round");
            return lst;
        }
        for (size_t i = 0; i < sh.size(); i++) ne[i] = pk[5 * i + 4];
        if (!c->virt && !c->host) return PEEL_OK;
        g[0] = g[1] = g[2] = g[3] = 0;
        for (size_t i = 0; i < sh.size(); i++) {
            g[0] += pk[5 * i]; g[1] += pk[5 * i + 1]; g[2] |= pk[5 * i + 2]; g[3] += pk[5 * i + 3];
        }
        if (lst != PEEL_OK) g[3] = 1;
        if (c->host) return comm_allreduce_sum(c, g, 4, dsum, s);
        return PEEL_OK;
    };

    ull g[4];
    if (!step(end_round(1, g)) || g[3]) return leave(g[3] != 0);
    if (g[2]) return PEEL_EINVAL;
    uint64_t alive_v = n;
    uint32_t t = 0;
    std::vector<ull> cnt_mat((size_t)P * P), rows((size_t)P * 9);
    while (g[0] > 0) {
        t++;
        alive_v -= g[0];
        if (t <= cap) {
            if (survivors) survivors[t - 1] = alive_v;
        }
        const int cur = t & 1, nxt = cur ^ 1;  // round t's entries live at parity (t&1): round 1 uses F[1]
        if (comm_fault(c, t) && lst == PEEL_OK) {
            set_cuda_error(cudaErrorUnknown, "PEEL_FAULT injected failure");
            lst = PEEL_ECUDA;
        }
        // kill: binned (decrements staged in the shard's bins) while the local frontier is large
        std::vector<char> binr(sh.size(), 0);
        uint32_t binmask = 0;
        for (size_t i = 0; i < sh.size(); i++) {
            const DShard &d = sh[i];
            binr[i] = d.binned && (double)ne[i] >= dist_bin_frac(d.v1 - d.v0) * (double)(d.v1 - d.v0);
            binmask |= (uint32_t)binr[i] << i;
        }
        // reset next-round counters and per-destination queues (ne[] came with the last sums),
        // and the binned shards' bin cursors and edge-sort counters
        dist_reset_kernel<<<(unsigned)sh.size(), 256, 0, s>>>(scs, nxt, binmask);
        cu(cudaGetLastError(), "reset");
        for (size_t i = 0; i < sh.size() && lst == PEEL_OK; i++) {
            DShard &d = sh[i];
            DKArgs a;
            a.edges = edges; a.n = n; a.m = m; a.P = P; a.p = d.q; a.k = k;
            for (int q = 0; q < 8; q++) a.lo[q] = q < P ? (uint32_t)shard_lo(n, P, q) : 0u;
            a.edges_vec = ((uintptr_t)edges & 15) == 0;
            a.v0 = d.v0; a.v1 = d.v1; a.nloc = nl_max;
            a.state = d.state; a.alive = d.alive;
            a.Fc = d.F[cur]; a.nE = ne[i]; a.Fn = d.F[nxt];
            a.send = d.send; a.ctl = d.ctl; a.par = nxt;
            if (binr[i]) {
                const ShardBinsView bv = shard_bins_view(n, m, R, d.v1 - d.v0, d.bins);
                // sort the local frontier by edge bin into the next-round buffer (free until
                // shard_apply writes F_{t+1} there)
                if (esort) {
                    if (!step(shard_edge_sort(d.F[cur], &d.ctl->ne[cur], a.nE, m, d.F[nxt], bv, s, true))) break;
                    a.Fc = d.F[nxt];
                }
                const size_t sm = dist_stage_smem(R, bv.nbins);
                const int kb = kill_blocks(false, sm);
                if (lst != PEEL_OK) break;
                ProfScope ps("dist_kill_binned", s);
                dist_kill_bin_kernel<R, false><<<num_sms() * (kb < 1 ? 1 : kb), DB, sm, s>>>(a, nullptr, 0, bv);
            } else {
                ProfScope ps("dist_kill", s);
                dist_kill_kernel<R><<<dgrid(a.nE), DB, 0, s>>>(a);
            }
        }
        cu(cudaGetLastError(), "kill launch");
        // count exchange: cnt_mat[src * P + dst], plus every rank's failure word -- ONE sync
        // (virtual: the shards' rows; ranks: one allgather of the 9-word rows nsend[8], fail)
        if (lst != PEEL_OK) mark_fail();
        bool peer_failed = false;
        if (c->virt) {  // shard i is shard q = i: the rows in shard order, one copy
            dist_rows_kernel<<<1, 9 * 8, 0, s>>>(scs, dsum + 8);
            cu(cudaMemcpyAsync(rows.data(), dsum + 8, sizeof(ull) * 9 * sh.size(), cudaMemcpyDeviceToHost, s), "rows");
            cu(cudaStreamSynchronize(s), "sync");
            if (lst != PEEL_OK) return lst;
        } else {
            if (!cu(cudaMemcpyAsync(dsum + 8 + 9 * c->rank, sh[0].ctl->nsend, sizeof(ull) * 9, cudaMemcpyDeviceToDevice, s), "rows")) {
                // the local row cannot be staged: still take part, with the failure word only
                std::vector<ull> fr(9, 0);
                fr[8] = 1;
                cudaMemcpyAsync(dsum + 8 + 9 * c->rank, fr.data(), sizeof(ull) * 9, cudaMemcpyHostToDevice, s);
            }
            peel_status sg;
            if (c->host) {
                std::vector<ull> mine(9);
                if (cudaMemcpyAsync(mine.data(), dsum + 8 + 9 * c->rank, sizeof(ull) * 9, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                    cudaStreamSynchronize(s) != cudaSuccess) {
                    cu(cudaGetLastError(), "rows");
                    mine.assign(9, 0);
                }
                if (lst != PEEL_OK) mine[8] = 1;
                sg = comm_allgather_u64(c, mine.data(), rows.data(), 9, dsum + 8, s);
            } else {
                // NCCL: gather the device rows in place, then one copy back
                sg = c->nccl ? PEEL_OK : comm_sync(c, s);  // aborted by the watchdog
                if (sg == PEEL_OK) {
                    ncclResult_t nr = ncclAllGather(dsum + 8 + 9 * c->rank, dsum + 8, 9, ncclUint64, c->nccl, s);
                    if (nr != ncclSuccess) { nccl_error(nr); sg = PEEL_ENCCL; }
                }
                if (sg == PEEL_OK) sg = comm_sync(c, s);  // before the copy back (see end_round)
                if (sg == PEEL_OK && (cudaMemcpyAsync(rows.data(), dsum + 8, sizeof(ull) * 9 * P, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                                      cudaStreamSynchronize(s) != cudaSuccess)) {
                    cu(cudaGetLastError(), "rows");
                    sg = PEEL_ECUDA;
                }
            }
            if (sg != PEEL_OK) return lst != PEEL_OK ? lst : sg;  // the transport itself failed
            for (int q = 0; q < P; q++) peer_failed |= rows[(size_t)q * 9 + 8] != 0;
            if (lst != PEEL_OK || peer_failed) return leave(peer_failed);
        }
        for (int q = 0; q < P; q++)
            for (int d = 0; d < P; d++) cnt_mat[(size_t)q * P + d] = rows[(size_t)q * 9 + d];
        // capacity: checked for EVERY receiver from the gathered matrix, so all ranks agree and
        // leave together (never from inside an open transport group)
        for (int dst = 0; dst < P; dst++) {
            ull tot = 0;
            for (int src = 0; src < P; src++)
                if (src != dst) tot += cnt_mat[(size_t)src * P + dst];
            if (tot > n) return PEEL_ENOMEM;
        }
        // payload: shard dst receives, from each src != dst, cnt[src][dst] ids into recv at running offsets
        std::vector<ull> nrecv(sh.size(), 0);
        if (c->virt) {  // every (src, dst) copy in one launch
            XPairs xp;
            xp.n = 0;
            ull mx = 0;
            for (int dst = 0; dst < P; dst++) {
                ull off = 0;
                for (int src = 0; src < P; src++) {
                    if (src == dst) continue;
                    const ull cntv = cnt_mat[(size_t)src * P + dst];
                    if (cntv) {
                        xp.src[xp.n] = sh[src].send + (uint64_t)dst * nl_max;
                        xp.dst[xp.n] = sh[dst].recv + off;
                        xp.cnt[xp.n] = cntv;
                        xp.n++;
                        mx = std::max(mx, cntv);
                    }
                    off += cntv;
                }
                nrecv[dst] = off;
            }
            if (xp.n) {
                const unsigned gx = (unsigned)std::min<ull>((mx + 255) / 256, (ull)num_sms() * 4);
                dist_xchg_kernel<<<dim3(gx, (unsigned)xp.n), 256, 0, s>>>(xp);
                cu(cudaGetLastError(), "virtual exchange");
            }
        } else {
            const int me = c->rank;
            std::vector<const char *> sp(P);
            std::vector<ull> sb(P), rb(P);
            ull off = 0;
            for (int q = 0; q < P; q++) {
                sp[q] = (const char *)(sh[0].send + (uint64_t)q * nl_max);
                sb[q] = q == me ? 0 : sizeof(uint32_t) * cnt_mat[(size_t)me * P + q];
                rb[q] = q == me ? 0 : sizeof(uint32_t) * cnt_mat[(size_t)q * P + me];
                off += rb[q] / sizeof(uint32_t);
            }
            peel_status sx = comm_alltoallv(c, sp.data(), sb.data(), (char *)sh[0].recv, rb.data(), s);
            if (sx != PEEL_OK) return sx;  // the transport failed (every rank sees its own error)
            nrecv[0] = off;
        }
        // receive (binned shards stage the received kills, then apply the round's bins)
        for (size_t i = 0; i < sh.size() && lst == PEEL_OK; i++) {
            DShard &d = sh[i];
            DKArgs a;
            a.edges = edges; a.n = n; a.m = m; a.P = P; a.p = d.q; a.k = k;
            for (int q = 0; q < 8; q++) a.lo[q] = q < P ? (uint32_t)shard_lo(n, P, q) : 0u;
            a.edges_vec = ((uintptr_t)edges & 15) == 0;
            a.v0 = d.v0; a.v1 = d.v1; a.nloc = nl_max;
            a.state = d.state; a.alive = d.alive;
            a.Fc = nullptr; a.nE = 0; a.Fn = d.F[nxt];
            a.send = d.send; a.ctl = d.ctl; a.par = nxt;
            if (binr[i]) {
                const ShardBinsView bv = shard_bins_view(n, m, R, d.v1 - d.v0, d.bins);
                if (nrecv[i]) {
                    const size_t sm = dist_stage_smem(R, bv.nbins);
                    const int kb = kill_blocks(true, sm);
                    if (lst != PEEL_OK) break;
                    ProfScope ps("dist_recv_binned", s);
                    dist_kill_bin_kernel<R, true><<<num_sms() * (kb < 1 ? 1 : kb), DB, sm, s>>>(a, d.recv, nrecv[i], bv);
                }
                step(shard_apply(d.v1 - d.v0, d.v0, k, d.state, d.F[nxt], bv, t, &d.ctl->nf[nxt], &d.ctl->ne[nxt], s));
                continue;
            }
            if (!nrecv[i]) continue;
            ProfScope ps("dist_recv", s);
            dist_recv_kernel<R><<<dgrid(nrecv[i]), DB, 0, s>>>(a, d.recv, nrecv[i]);
        }
        cu(cudaGetLastError(), "receive launch");
        if (lst != PEEL_OK && c->virt) return lst;
        if (!step(end_round(nxt, g)) || g[3]) return leave(g[3] != 0);
        if (t <= cap && killed) killed[t - 1] = g[1];
    }
    *rounds = t;
    for (auto &d : sh) {
        uint8_t *mk = core_mask + (c->virt ? d.v0 : 0);
        ProfScope ps("dist_mask", s);
        dist_mask_kernel<<<dgrid(d.v1 - d.v0), DB, 0, s>>>(d.state, d.v1 - d.v0, k, mk);
    }
    PEEL_CUDA(cudaGetLastError());
    PEEL_CUDA(cudaStreamSynchronize(s));
    prof_collect();
    return t > cap ? PEEL_ETRUNC : PEEL_OK;
}

extern "C" peel_status peel_kcore_dist(peel_comm *c, const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r,
                                       uint32_t k, uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors,
                                       uint64_t *killed, uint32_t cap, void *workspace, size_t ws_bytes,
                                       void *stream) {
    if (!c) return PEEL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    size_t need = peel_kcore_dist_workspace_bytes(c, n, m, r, k);
    peel_status v = PEEL_OK;
    if (!need || !rounds || !workspace || (m && !edges) || !core_mask) v = PEEL_EINVAL;
    else if (ws_bytes < need) v = PEEL_ENOMEM;
    v = comm_agree(c, v, s);  // every rank leaves together if any rank rejects its arguments
    if (v != PEEL_OK) return v;
    prof_begin_call();
    char *ws = (char *)workspace;
    switch (r) {
        case 2: return run_dist<2>(c, edges, n, m, k, core_mask, rounds, survivors, killed, cap, ws, s);
        case 3: return run_dist<3>(c, edges, n, m, k, core_mask, rounds, survivors, killed, cap, ws, s);
        case 4: return run_dist<4>(c, edges, n, m, k, core_mask, rounds, survivors, killed, cap, ws, s);
        case 5: return run_dist<5>(c, edges, n, m, k, core_mask, rounds, survivors, killed, cap, ws, s);
        case 6: return run_dist<6>(c, edges, n, m, k, core_mask, rounds, survivors, killed, cap, ws, s);
        case 7: return run_dist<7>(c, edges, n, m, k, core_mask, rounds, survivors, killed, cap, ws, s);
        case 8: return run_dist<8>(c, edges, n, m, k, core_mask, rounds, survivors, killed, cap, ws, s);
    }
    return PEEL_EINVAL;
}
