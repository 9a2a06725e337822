// iblt.cu -- IBLT insert/delete and round-synchronous recovery on sm_100a
// (P:474-513).
//
// Cells are 16 B {u32 count, u32 hashSum, u64 keySum}: two cells per 32-byte
// sector, the three fields of one cell in one sector.  Insert/delete: one
// thread per key, r x 3 atomics.  Recovery is the 2-core peel of
// the IBLT's hypergraph, one cooperative persistent kernel:
//
//   round 1   scan all C cells; pure cells -> frontier entries (cell, key)
//             (the key is snapshotted) + round-start "pure" bitmap.
//   phase A   for each entry (c, x): x is recovered by this entry iff c is
//             the LOWEST-index cell among h_1(x)..h_r(x) that was pure at round
//             start (each round-start-pure cell holding x holds only x, so the
//             owner is unique: exactly-once deletion without the paper's r
//             serial subtable steps).  The owner XOR-deletes x from
//             its r cells with atomics; a cell whose count drops
//             2 -> 1 becomes a candidate (deduplicated by a bitmap).
//   phase B   clear the round's pure bits; re-test candidates for purity
//             (a candidate may have dropped to 0 in the same round) and emit
//             the next frontier.
//   stop      at the first round with an empty frontier.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "iblt_common.cuh"

namespace peel {

static constexpr uint32_t ISTAT_CAP = 65536;
static constexpr int IB_BLOCK = 256;



struct IbltCtl {
    ull fcnt[3];   // frontier sizes, F_t uses fcnt[(t-1)%3]
    ull ccnt[2];   // candidate-list sizes, round t appends ccnt[t%2]
    ull nrec;      // keys recovered so far
    ull rounds;
    ull scnt[16];  // subtable mode: list lengths [subtable j][round parity b] at j * 2 + b
    uint32_t nonzero;
    uint32_t trunc;  // the round limit (ISTAT_CAP rounds / subtable steps) stopped recovery
};

struct ILayout {
    size_t cells, ctl, per_round, rtime, pure0, pure1, cand, F0, F1, clist, total;
};

static inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static ILayout ilayout(uint64_t C) {
    ILayout L;
    size_t o = 0;
    L.cells = o; o += al(sizeof(Cell) * C);
    L.ctl = o; o += al(sizeof(IbltCtl));
    L.per_round = o; o += al(sizeof(ull) * (ISTAT_CAP + 1));
    L.rtime = o; o += al(sizeof(ull) * (ISTAT_CAP + 2));  // %globaltimer at each round start (profiling)
    L.pure0 = o; o += al(sizeof(uint32_t) * ((C + 31) / 32));
    L.pure1 = o; o += al(sizeof(uint32_t) * ((C + 31) / 32));
    L.cand = o; o += al(sizeof(uint32_t) * ((C + 31) / 32));
    L.F0 = o; o += al(sizeof(ulonglong2) * C);
    L.F1 = o; o += al(sizeof(ulonglong2) * C);
    L.clist = o; o += al(sizeof(uint32_t) * C);
    L.total = o;
    return L;
}

// one pass of an insert/delete: the r cells of every key, restricted to cells in [lo, hi)
// (a table larger than ~half the L2 is updated in several passes over the keys, each
// pass's cell range L2-resident)
template <int R>
__global__ void __launch_bounds__(256) iblt_update_kernel(Cell *cells, ull C, ull seed_h, ull seed_c,
                                                          const ull *__restrict__ keys, ull nkeys,
                                                          uint32_t delta, bool subt, uint32_t lo, uint32_t hi,
                                                          uint32_t blog) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nkeys; i += (ull)gridDim.x * blockDim.x) {
        const ull x = __ldg(keys + i);
        uint32_t c[R];
        key_cells<R>(x, C, seed_h, subt, c, blog);
        const uint32_t h = checksum(x, seed_c);
        #pragma unroll
        for (int j = 0; j < R; j++) {
            if (c[j] < lo || c[j] >= hi) continue;
            Cell *p = cells + c[j];
            atomicAdd(&p->count, delta);
            atomicXor(&p->keySum, x);
            atomicXor(&p->hashSum, h);
        }
    }
}

template <int R>
__global__ void __launch_bounds__(256) iblt_edges_kernel(ull C, ull seed_h, const ull *__restrict__ keys,
                                                         ull nkeys, uint32_t *edges, bool subt, uint32_t blog) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nkeys; i += (ull)gridDim.x * blockDim.x) {
        uint32_t c[R];
        key_cells<R>(__ldg(keys + i), C, seed_h, subt, c, blog);
        #pragma unroll
        for (int j = 0; j < R; j++) edges[i * R + j] = c[j];
    }
}

struct IPeelArgs {
    Cell *cells;
    ull C, seed_h, seed_c;
    IbltCtl *ctl;
    ull *per_round;
    ull *rtime;
    uint32_t *pure[2];  // round-start pure bitmaps: F_t's bits live in pure[(t-1)&1]
    uint32_t *cand;
    ulonglong2 *F[2];   // frontier entries (cell, key snapshot)
    uint32_t *clist;
    ull *out;
    int8_t *out_sign;   // signed recovery: +1 / -1 per recovered key
    ull cap_keys;
    bool subt;          // subtable hashing
    uint32_t blog;      // blocked hashing: log2 block size, 0 = off
    bool insert_only;   // every count is the true number of keys in its cell (no delete/subtract)
    ull ninserted;      // insert-only: keys inserted since the build (complete iff all recovered)
};


// signed tables (set difference): pure = count +1 or -1 with a matching checksum, and cell c
// is one of the key's cells (R26, R28); returns +1 / -1, or 0 if not pure.  Unsigned recovery
// accepts only count == +1.
template <int R, bool SIGNED>
__device__ __forceinline__ int pure_sign(const Cell &v, uint32_t c, const IPeelArgs &a) {
    const bool cnt = SIGNED ? (v.count == 1u || v.count == 0xFFFFFFFFu) : (v.count == 1u);
    if (!cnt || v.hashSum != checksum(v.keySum, a.seed_c)) return 0;
    // in an insert-only table a count-1 cell holds exactly one inserted key, which hashes to it:
    // the R28 test can only pass, and is skipped
    if (!(!SIGNED && a.insert_only) && !cell_of_key<R>(c, v.keySum, a.C, a.seed_h, a.subt, a.blog)) return 0;
    return v.count == 1u ? 1 : -1;
}

// w[0, nwords) = 0 over the whole grid (w is 256-byte aligned: 16-byte stores, then the tail)
__device__ __forceinline__ void zero_words(uint32_t *w, ull nwords, ull tid, ull nthr) {
    const ull n4 = nwords / 4;
    for (ull i = tid; i < n4; i += nthr) __stcg(reinterpret_cast<uint4 *>(w) + i, make_uint4(0u, 0u, 0u, 0u));
    for (ull i = n4 * 4 + tid; i < nwords; i += nthr) w[i] = 0u;
}

static constexpr int IQ = 2 * IB_BLOCK;
typedef BlockQueueT<ulonglong2, IQ, IB_BLOCK> EntQ;
typedef BlockQueueT<ull, IQ, IB_BLOCK> KeyQ;
typedef BlockQueueT<uint32_t, IQ, IB_BLOCK> CellQ;

// entry.x = cell | (negative sign) << 32, entry.y = key snapshot
// 5 resident blocks per SM (48 registers; shared queues 36 KB per block): C2 peel 1.38 ms at
// 4 blocks (64 registers), 1.35 ms at 5; 6 and 8 blocks spill or lose to the smaller queues
// of registers: 1.60 / 1.64 ms
template <int R, bool SIGNED>
__global__ void __launch_bounds__(IB_BLOCK, 5) iblt_peel_kernel(IPeelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ EntQ qe;
    __shared__ EntQ qk;  // recovered (key, sign)
    __shared__ CellQ qc;
    IbltCtl *ctl = a.ctl;
    bq_init(qe); bq_init(qk); bq_init(qc);
    __syncthreads();
    const ull tid = blockIdx.x * (ull)blockDim.x + threadIdx.x;
    const ull nthr = (ull)gridDim.x * blockDim.x;
    const ull stride = (ull)gridDim.x * IB_BLOCK;
    int slot = 0;
    auto write_key = [&](ull i, ulonglong2 v) {
        a.out[i] = v.x;
        if (SIGNED) a.out_sign[i] = (int8_t)(v.y ? -1 : 1);
    };

    // ---- round 1: every pure cell ("a single thread to each cell") ----
    for (ull base = (ull)blockIdx.x * IB_BLOCK; base < a.C; base += stride) {
        const ull c = base + threadIdx.x;
        if (c < a.C) {
            Cell v = ld_cell_cg(a.cells + c);
            const int sg = pure_sign<R, SIGNED>(v, (uint32_t)c, a);
            if (sg) {
                bq_push(qe, slot, make_ulonglong2(c | ((ull)(sg < 0) << 32), v.keySum), a.F[0], &ctl->fcnt[0]);
                atomicOr(a.pure[0] + (c >> 5), 1u << (c & 31));
            }
        }
        bq_flush(qe, slot, a.F[0], &ctl->fcnt[0]);
        slot ^= 1;
    }
    grid.sync();

    uint32_t t = 1;
    for (;;) {
        const ull nF = ld_cg_u64(&ctl->fcnt[(t - 1) % 3]);
        if (nF == 0) break;
        if (t > ISTAT_CAP) {  // round limit (R28: forged signed tables can cycle)
            if (tid == 0) ctl->trunc = 1u;
            break;
        }
        if (tid == 0) {
            ctl->fcnt[(t + 1) % 3] = 0;
            if (t <= ISTAT_CAP) a.rtime[t - 1] = globaltimer();
        }
        const ulonglong2 *Fc = a.F[(t - 1) & 1];
        ull *ccnt = &ctl->ccnt[t & 1];
        const uint32_t *pure_cur = a.pure[(t - 1) & 1];
        ull recovered = 0;
        // ---- phase A: owner rule, XOR-delete, candidates ----
        for (ull base = (ull)blockIdx.x * IB_BLOCK; base < nF; base += stride) {
            const ull i = base + threadIdx.x;
            if (i < nF) {
                const ulonglong2 ent = __ldcg(Fc + i);
                const uint32_t c = (uint32_t)ent.x;
                const bool neg = (ent.x >> 32) != 0;
                const ull x = ent.y;
                uint32_t h[R];
                key_cells<R>(x, a.C, a.seed_h, a.subt, h, a.blog);
                // owner rule: c is one of x's cells and none of x's cells of lower index was
                // pure at round start (only those pure bits are loaded, together)
                uint32_t pw[R];
                #pragma unroll
                for (int j = 0; j < R; j++) pw[j] = h[j] < c ? ld_cg_u32(pure_cur + (h[j] >> 5)) : 0u;
                bool owner = false;
                #pragma unroll
                for (int j = 0; j < R; j++) owner |= h[j] == c;
                #pragma unroll
                for (int j = 0; j < R; j++)
                    if (h[j] < c && (pw[j] >> (h[j] & 31) & 1u)) owner = false;
                if (owner) {
                    recovered++;
                    // <= one push per thread per iteration < IQ: the queue never takes its overflow path
                    bq_push(qk, slot, make_ulonglong2(x, neg ? 1ull : 0ull), (ulonglong2 *)nullptr, &ctl->nrec);
                    const uint32_t hx = checksum(x, a.seed_c);
                    const uint32_t delta = neg ? 1u : 0xFFFFFFFFu;  // remove: count -= sign
                    // the r count atomics are issued before any result is used.  In an
                    // insert-only table the round-start-pure cell c holds x alone, and no
                    // other key recovered this round can be in it: x's deletion leaves it
                    // zero, a plain 16-byte store instead of three atomics.
                    uint32_t now[R];
                    #pragma unroll
                    for (int j = 0; j < R; j++) {
                        Cell *p = a.cells + h[j];
                        if (!SIGNED && a.insert_only && h[j] == c) {
                            __stcg(reinterpret_cast<uint4 *>(p), make_uint4(0u, 0u, 0u, 0u));
                            now[j] = 0u;
                            continue;
                        }
                        now[j] = atomicAdd(&p->count, delta) + delta;
                        atomicXor(&p->keySum, x);
                        atomicXor(&p->hashSum, hx);
                    }
                    #pragma unroll
                    for (int j = 0; j < R; j++)
                        if (now[j] == 1u || (SIGNED && now[j] == 0xFFFFFFFFu)) {
                            const uint32_t bit = 1u << (h[j] & 31);
                            if (!(atomicOr(a.cand + (h[j] >> 5), bit) & bit)) bq_push(qc, slot, h[j], a.clist, ccnt);
                        }
                }
            }
            bq_flush_with(qk, slot, &ctl->nrec, a.cap_keys, write_key);
            bq_flush(qc, slot, a.clist, ccnt);
            slot ^= 1;
        }
        block_add<IB_BLOCK>(&a.per_round[t <= ISTAT_CAP ? t - 1 : ISTAT_CAP], recovered);
        grid.sync();
        // ---- phase B: retire this round's pure bits, re-test candidates ----
        // pure[(t-1)&1] holds exactly F_t's bits and cand exactly this round's candidates:
        // a large round zeroes the whole bitmap with coalesced stores (C/8 bytes) instead of
        // one random atomicAnd per entry
        const ull nwords = (a.C + 31) / 32;
        if (nF * 8 >= nwords) zero_words(a.pure[(t - 1) & 1], nwords, tid, nthr);
        else
            for (ull i = tid; i < nF; i += nthr) {
                const uint32_t c = (uint32_t)__ldcg(&Fc[i].x);
                atomicAnd(a.pure[(t - 1) & 1] + (c >> 5), ~(1u << (c & 31)));
            }
        if (tid == 0) ctl->ccnt[(t + 1) & 1] = 0;
        const ull nC = ld_cg_u64(ccnt);
        const bool cand_bulk = nC * 8 >= nwords;
        if (cand_bulk) zero_words(a.cand, nwords, tid, nthr);
        ulonglong2 *Fn = a.F[t & 1];
        ull *fn = &ctl->fcnt[t % 3];
        uint32_t *pure_next = a.pure[t & 1];
        for (ull base = (ull)blockIdx.x * IB_BLOCK; base < nC; base += stride) {
            const ull i = base + threadIdx.x;
            if (i < nC) {
                const uint32_t c = ld_cg_u32(a.clist + i);
                if (!cand_bulk) atomicAnd(a.cand + (c >> 5), ~(1u << (c & 31)));
                Cell v = ld_cell_cg(a.cells + c);
                const int sg = pure_sign<R, SIGNED>(v, c, a);
                if (sg) {
                    bq_push(qe, slot, make_ulonglong2(c | ((ull)(sg < 0) << 32), v.keySum), Fn, fn);
                    atomicOr(pure_next + (c >> 5), 1u << (c & 31));
                }
            }
            bq_flush(qe, slot, Fn, fn);
            slot ^= 1;
        }
        grid.sync();
        t++;
    }
    if (tid == 0) {
        ctl->rounds = t - 1;
        if (t <= ISTAT_CAP) a.rtime[t - 1] = globaltimer();
    }
    // ---- complete iff every cell is zero ----
    // An insert-only table is the multiset sum of its N inserted keys, and recovery removed
    // exactly the recovered ones: every cell is zero iff all N were recovered -- no scan of the
    // C cells (C2: 160 MB)
    if (!SIGNED && a.insert_only) {
        if (tid == 0 && ld_cg_u64(&ctl->nrec) != a.ninserted) ctl->nonzero = 1u;
        return;
    }
    uint32_t nz = 0;
    for (ull c = tid; c < a.C; c += nthr) {
        Cell v = ld_cell_cg(a.cells + c);
        nz |= (v.count | v.hashSum) != 0u || v.keySum != 0ull;
    }
    if (__any_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) atomicOr(&ctl->nonzero, 1u);
}

// ---- subtable recovery: each round iterates the r subtables serially --------
// Subtable j's step processes the list of subtable-j cells that may be pure: each is
// re-tested and, if pure, its key recovered and deleted from its r cells (one per
// subtable, so a key is found in at most one pure cell of subtable j: exactly once without
// any owner rule).  A cell of subtable j' whose count drops 2 -> 1 joins subtable j''s list
// for this round (j' > j) or the next (j' < j); subtable j's own cells only drop 1 -> 0.
// Lists: (uint32 *)F0 + b C + j C/r, b = round parity.
static constexpr int SQ = 2 * IB_BLOCK;
typedef BlockQueueT<uint32_t, SQ, IB_BLOCK> SCellQ;

template <int R>
__global__ void __launch_bounds__(IB_BLOCK) iblt_subtable_peel_kernel(IPeelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ SCellQ qs[R];
    __shared__ KeyQ qk;
    IbltCtl *ctl = a.ctl;
    #pragma unroll
    for (int j = 0; j < R; j++) bq_init(qs[j]);
    bq_init(qk);
    __syncthreads();
    const ull tid = blockIdx.x * (ull)blockDim.x + threadIdx.x;
    const ull nthr = (ull)gridDim.x * blockDim.x;
    const ull stride = (ull)gridDim.x * IB_BLOCK;
    const ull cs = a.C / R;
    uint32_t *L0 = reinterpret_cast<uint32_t *>(a.F[0]);
    auto list = [&](uint32_t j, uint32_t b) { return L0 + (ull)b * a.C + (ull)j * cs; };
    int slot = 0;
    // round 1's lists: every pure cell, in its subtable's list (parity 0)
    for (ull base = (ull)blockIdx.x * IB_BLOCK; base < a.C; base += stride) {
        const ull c = base + threadIdx.x;
        bool p = false;
        if (c < a.C) {
            Cell v = ld_cell_cg(a.cells + c);
            p = is_pure(v, a.seed_c) && cell_of_key<R>((uint32_t)c, v.keySum, a.C, a.seed_h, true, 0u);
            if (p) atomicOr(a.cand + (c >> 5), 1u << (c & 31));
        }
        const uint32_t jc = (uint32_t)(c / cs);
        #pragma unroll
        for (int j = 0; j < R; j++)
            if (p && jc == (uint32_t)j) bq_push(qs[j], slot, (uint32_t)c, list(j, 0), &ctl->scnt[j * 2 + 0]);
        #pragma unroll
        for (int j = 0; j < R; j++) bq_flush(qs[j], slot, list(j, 0), &ctl->scnt[j * 2 + 0]);
        slot ^= 1;
    }
    grid.sync();
    uint32_t flat = 0, last = 0;
    for (uint32_t i = 0;; i++) {
        bool any = false;
        const uint32_t b = i & 1u;
        if (flat + (uint32_t)R > ISTAT_CAP) {  // step limit, as the oracle's
            if (tid == 0) ctl->trunc = 1u;
            break;
        }
        #pragma unroll 1
        for (uint32_t j = 0; j < (uint32_t)R; j++) {
            flat++;
            const ull nL = ld_cg_u64(&ctl->scnt[j * 2 + b]);
            const uint32_t *Lc = list(j, b);
            ull recovered = 0;
            for (ull base = (ull)blockIdx.x * IB_BLOCK; base < nL; base += stride) {
                const ull q = base + threadIdx.x;
                uint32_t h[R];
                bool cand[R];
                ull x = 0;
                #pragma unroll
                for (int jj = 0; jj < R; jj++) cand[jj] = false;
                if (q < nL) {
                    const uint32_t c = ld_cg_u32(Lc + q);
                    atomicAnd(a.cand + (c >> 5), ~(1u << (c & 31)));
                    Cell v = ld_cell_cg(a.cells + c);
                    if (is_pure(v, a.seed_c) && cell_of_key<R>(c, v.keySum, a.C, a.seed_h, true, 0u)) {
                        x = v.keySum;
                        recovered++;
                        bq_push(qk, slot, x, a.out, &ctl->nrec);
                        key_cells<R>(x, a.C, a.seed_h, true, h);
                        const uint32_t hx = checksum(x, a.seed_c);
                        #pragma unroll
                        for (int jj = 0; jj < R; jj++) {
                            Cell *p = a.cells + h[jj];
                            const uint32_t old = atomicAdd(&p->count, 0xFFFFFFFFu);
                            atomicXor(&p->keySum, x);
                            atomicXor(&p->hashSum, hx);
                            if (old == 2u && (uint32_t)jj != j) {
                                const uint32_t bit = 1u << (h[jj] & 31);
                                cand[jj] = !(atomicOr(a.cand + (h[jj] >> 5), bit) & bit);
                            }
                        }
                    }
                }
                #pragma unroll
                for (int jj = 0; jj < R; jj++) {
                    const uint32_t bb = (uint32_t)jj > j ? b : (b ^ 1u);
                    if (cand[jj]) bq_push(qs[jj], slot, h[jj], list(jj, bb), &ctl->scnt[jj * 2 + bb]);
                }
                #pragma unroll
                for (int jj = 0; jj < R; jj++) {
                    const uint32_t bb = (uint32_t)jj > j ? b : (b ^ 1u);
                    bq_flush(qs[jj], slot, list(jj, bb), &ctl->scnt[jj * 2 + bb]);
                }
                bq_flush(qk, slot, a.out, &ctl->nrec, a.cap_keys);
                slot ^= 1;
            }
            block_add<IB_BLOCK>(&a.per_round[flat <= ISTAT_CAP ? flat - 1 : ISTAT_CAP], recovered);
            grid.sync();
            const ull got = ld_cg_u64(&a.per_round[flat <= ISTAT_CAP ? flat - 1 : ISTAT_CAP]);
            if (tid == 0) ctl->scnt[j * 2 + b] = 0;  // consumed; next appended a round later
            if (got) { any = true; last = flat; }
        }
        if (!any) break;
    }
    if (tid == 0) ctl->rounds = last;
    uint32_t nz = 0;
    for (ull c = tid; c < a.C; c += nthr) {
        Cell v = ld_cell_cg(a.cells + c);
        nz |= (v.count | v.hashSum) != 0u || v.keySum != 0ull;
    }
    if (__any_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) atomicOr(&ctl->nonzero, 1u);
}

static unsigned grid_for(ull work, int per_sm = 16) {
    ull blocks = (work + 255) / 256;
    ull cap = (ull)num_sms() * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    return (unsigned)blocks;
}

}  // namespace peel

using namespace peel;

struct peel_iblt {
    ull C;
    uint32_t r;
    bool subt;  // IBLT_FLAG_SUBTABLES
    uint32_t blog;  // IBLT_FLAG_BLOCKED: log2 cells per block (0: plain hashing)
    mutable bool insert_only;  // no delete, no subtract, no raw cell access since the build
    ull ninserted;             // keys inserted since the build
    ull seed, seed_h, seed_c;
    char *mem;
    ILayout L;
};

static ull host_mix64(ull z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

extern "C" size_t iblt_mem_bytes(uint64_t cells, uint32_t r) {
    if (r < 2 || r > 8 || cells < r || cells >= (1ull << 32)) return 0;
    return ilayout(cells).total;
}

extern "C" peel_status iblt_build_ex(uint64_t cells, uint32_t r, uint64_t seed, uint32_t flags, void *mem,
                                     size_t mem_bytes, void *stream, peel_iblt **out) {
    if (!out || !mem || r < 2 || r > 8 || cells < r || cells >= (1ull << 32)) return PEEL_EINVAL;
    if ((flags & IBLT_FLAG_SUBTABLES) && cells % r) return PEEL_EINVAL;
    uint32_t blog = 0;
    if (flags & IBLT_FLAG_BLOCKED) {
        blog = IBLT_BLOCK_LOG(flags) ? IBLT_BLOCK_LOG(flags) : 16u;
        if ((flags & IBLT_FLAG_SUBTABLES) || blog < 4 || blog > 30 || cells % (1ull << blog) || (1ull << blog) < r)
            return PEEL_EINVAL;
    }
    if (((uintptr_t)mem & 15) != 0) return PEEL_EINVAL;
    ILayout L = ilayout(cells);
    if (mem_bytes < L.total) return PEEL_ENOMEM;
    cudaStream_t s = (cudaStream_t)stream;
    prof_begin_call();
    PEEL_CUDA(cudaMemsetAsync(mem, 0, sizeof(Cell) * cells, s));
    peel_iblt *t = new peel_iblt;
    t->C = cells;
    t->r = r;
    t->subt = (flags & IBLT_FLAG_SUBTABLES) != 0;
    t->blog = blog;
    t->insert_only = true;
    t->ninserted = 0;
    t->seed = seed;
    const ull G = 0x9E3779B97F4A7C15ull;
    t->seed_h = host_mix64((seed ^ 0x6A09E667F3BCC909ull) + G);
    t->seed_c = host_mix64((seed ^ 0xBB67AE8584CAA73Bull) + G);
    t->mem = (char *)mem;
    t->L = L;
    *out = t;
    return PEEL_OK;
}

extern "C" peel_status iblt_build(uint64_t cells, uint32_t r, uint64_t seed, void *mem, size_t mem_bytes,
                                  void *stream, peel_iblt **out) {
    return iblt_build_ex(cells, r, seed, 0u, mem, mem_bytes, stream, out);
}

static peel_status iblt_update(peel_iblt *t, const uint64_t *keys, uint64_t nkeys, uint32_t delta,
                               void *stream) {
    if (!t) return PEEL_EINVAL;
    if (nkeys == 0) return PEEL_OK;
    if (!keys) return PEEL_EINVAL;
    if (delta != 1u) t->insert_only = false;
    else t->ninserted += nkeys;
    cudaStream_t s = (cudaStream_t)stream;
    prof_begin_call();
    Cell *cells = (Cell *)(t->mem + t->L.cells);
    unsigned g = grid_for(nkeys);
#ifndef PEEL_IBLT_PASS_BYTES
#define PEEL_IBLT_PASS_BYTES (64ull << 20)
#endif
    // at most 8 passes: every pass re-reads and re-hashes all keys (C = 2^28 cells: 67 passes of
    // 64 MB 110 ms, 9 of 512 MB 29 ms, 1 pass 39 ms; C2's 160 MB table: 3 passes 0.40 ms, 1 pass 0.70)
    const uint64_t npass = std::min<uint64_t>(8, (t->C * sizeof(Cell) + PEEL_IBLT_PASS_BYTES - 1) / PEEL_IBLT_PASS_BYTES);
    ProfScope ps(delta == 1u ? "iblt_insert" : "iblt_delete", s);
    for (uint64_t q = 0; q < npass; q++) {
        const uint32_t lo = (uint32_t)(q * t->C / npass), hi = (uint32_t)((q + 1) * t->C / npass);
        switch (t->r) {
            case 2: iblt_update_kernel<2><<<g, 256, 0, s>>>(cells, t->C, t->seed_h, t->seed_c, (const ull *)keys, nkeys, delta, t->subt, lo, hi, t->blog); break;
            case 3: iblt_update_kernel<3><<<g, 256, 0, s>>>(cells, t->C, t->seed_h, t->seed_c, (const ull *)keys, nkeys, delta, t->subt, lo, hi, t->blog); break;
            case 4: iblt_update_kernel<4><<<g, 256, 0, s>>>(cells, t->C, t->seed_h, t->seed_c, (const ull *)keys, nkeys, delta, t->subt, lo, hi, t->blog); break;
            case 5: iblt_update_kernel<5><<<g, 256, 0, s>>>(cells, t->C, t->seed_h, t->seed_c, (const ull *)keys, nkeys, delta, t->subt, lo, hi, t->blog); break;
            case 6: iblt_update_kernel<6><<<g, 256, 0, s>>>(cells, t->C, t->seed_h, t->seed_c, (const ull *)keys, nkeys, delta, t->subt, lo, hi, t->blog); break;
            case 7: iblt_update_kernel<7><<<g, 256, 0, s>>>(cells, t->C, t->seed_h, t->seed_c, (const ull *)keys, nkeys, delta, t->subt, lo, hi, t->blog); break;
            case 8: iblt_update_kernel<8><<<g, 256, 0, s>>>(cells, t->C, t->seed_h, t->seed_c, (const ull *)keys, nkeys, delta, t->subt, lo, hi, t->blog); break;
        }
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}

extern "C" peel_status iblt_insert(peel_iblt *t, const uint64_t *keys, uint64_t nkeys, void *stream) {
    return iblt_update(t, keys, nkeys, 1u, stream);
}

extern "C" peel_status iblt_delete(peel_iblt *t, const uint64_t *keys, uint64_t nkeys, void *stream) {
    return iblt_update(t, keys, nkeys, 0xFFFFFFFFu, stream);
}

template <int R>
static peel_status run_iblt_peel(peel_iblt *t, IPeelArgs &a, bool sgn, cudaStream_t s) {
    void *kern = t->subt ? (void *)iblt_subtable_peel_kernel<R>
                         : (sgn ? (void *)iblt_peel_kernel<R, true> : (void *)iblt_peel_kernel<R, false>);
    int per_sm = 0;
    PEEL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, IB_BLOCK, 0));
    if (per_sm < 1) per_sm = 1;
    unsigned grid = (unsigned)(num_sms() * per_sm);
    const ull want = (t->C + IB_BLOCK - 1) / IB_BLOCK;  // small tables: cheaper grid barriers
    if (want < grid) grid = (unsigned)(want < (ull)num_sms() ? num_sms() : want);
    void *args[] = {&a};
    ProfScope ps(t->subt ? "iblt_subtable_peel" : (sgn ? "iblt_peel_signed_rounds" : "iblt_peel_rounds"), s);
    PEEL_CUDA(cudaLaunchCooperativeKernel(kern, grid, IB_BLOCK, args, 0, s));
    return PEEL_OK;
}

static peel_status iblt_peel_impl(peel_iblt *t, uint64_t *out_keys, int8_t *out_sign, uint64_t cap_keys,
                                  uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round, uint32_t cap,
                                  int *complete, void *stream) {
    const bool sgn = out_sign != nullptr;
    if (!t || !nrecovered || !rounds || (cap_keys && !out_keys)) return PEEL_EINVAL;
    if (sgn && t->subt) return PEEL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    prof_begin_call();
    const ILayout &L = t->L;
    char *m = t->mem;
    // zero control, per-round stats and both bitmaps (contiguous)
    PEEL_CUDA(cudaMemsetAsync(m + L.ctl, 0, L.F0 - L.ctl, s));
    IPeelArgs a;
    memset(&a, 0, sizeof a);
    a.cells = (Cell *)(m + L.cells);
    a.C = t->C;
    a.seed_h = t->seed_h;
    a.seed_c = t->seed_c;
    a.ctl = (IbltCtl *)(m + L.ctl);
    a.per_round = (ull *)(m + L.per_round);
    a.rtime = (ull *)(m + L.rtime);
    a.pure[0] = (uint32_t *)(m + L.pure0);
    a.pure[1] = (uint32_t *)(m + L.pure1);
    a.cand = (uint32_t *)(m + L.cand);
    a.F[0] = (ulonglong2 *)(m + L.F0);
    a.F[1] = (ulonglong2 *)(m + L.F1);
    a.clist = (uint32_t *)(m + L.clist);
    a.out = (ull *)out_keys;
    a.out_sign = out_sign;
    a.cap_keys = cap_keys;
    a.subt = t->subt;
    a.blog = t->blog;
    a.insert_only = t->insert_only;
    a.ninserted = t->ninserted;
    peel_status st = PEEL_EINVAL;
    switch (t->r) {
        case 2: st = run_iblt_peel<2>(t, a, sgn, s); break;
        case 3: st = run_iblt_peel<3>(t, a, sgn, s); break;
        case 4: st = run_iblt_peel<4>(t, a, sgn, s); break;
        case 5: st = run_iblt_peel<5>(t, a, sgn, s); break;
        case 6: st = run_iblt_peel<6>(t, a, sgn, s); break;
        case 7: st = run_iblt_peel<7>(t, a, sgn, s); break;
        case 8: st = run_iblt_peel<8>(t, a, sgn, s); break;
    }
    if (st != PEEL_OK) return st;
    IbltCtl h;
    PEEL_CUDA(cudaMemcpyAsync(&h, a.ctl, sizeof h, cudaMemcpyDeviceToHost, s));
    PEEL_CUDA(cudaStreamSynchronize(s));
    prof_collect();
    if (prof_enabled() && !t->subt && h.rounds) {
        const uint64_t nt = (h.rounds < ISTAT_CAP ? h.rounds : ISTAT_CAP - 1) + 1;
        std::vector<ull> rt(nt);
        PEEL_CUDA(cudaMemcpy(rt.data(), a.rtime, sizeof(ull) * nt, cudaMemcpyDeviceToHost));
        std::vector<double> ms(nt - 1);
        for (uint64_t i = 0; i + 1 < nt; i++) ms[i] = (rt[i + 1] - rt[i]) * 1e-6;
        prof_set_rounds(ms);
    }
    *nrecovered = h.nrec;
    *rounds = (uint32_t)h.rounds;
    if (complete) *complete = h.nonzero ? 0 : 1;
    uint64_t nstore = h.rounds < cap ? h.rounds : cap;
    if (nstore > ISTAT_CAP) nstore = ISTAT_CAP;
    if (per_round && nstore)
        PEEL_CUDA(cudaMemcpy(per_round, a.per_round, sizeof(ull) * nstore, cudaMemcpyDeviceToHost));
    if (h.nrec > cap_keys || h.rounds > cap || h.rounds > ISTAT_CAP || h.trunc) return PEEL_ETRUNC;
    return PEEL_OK;
}

extern "C" peel_status iblt_peel(peel_iblt *t, uint64_t *out_keys, uint64_t cap_keys, uint64_t *nrecovered,
                                 uint32_t *rounds, uint64_t *per_round, uint32_t cap, int *complete,
                                 void *stream) {
    return iblt_peel_impl(t, out_keys, nullptr, cap_keys, nrecovered, rounds, per_round, cap, complete, stream);
}

extern "C" peel_status iblt_peel_signed(peel_iblt *t, uint64_t *out_keys, int8_t *out_sign, uint64_t cap_keys,
                                        uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round, uint32_t cap,
                                        int *complete, void *stream) {
    if (!out_sign && cap_keys) return PEEL_EINVAL;
    static int8_t dummy;
    return iblt_peel_impl(t, out_keys, out_sign ? out_sign : &dummy, cap_keys, nrecovered, rounds, per_round, cap,
                          complete, stream);
}

// a <- a - b cell-wise: count subtracts, key and checksum fields XOR
__global__ void __launch_bounds__(256) iblt_subtract_kernel(Cell *a, const Cell *__restrict__ b, ull C) {
    for (ull c = blockIdx.x * (ull)blockDim.x + threadIdx.x; c < C; c += (ull)gridDim.x * blockDim.x) {
        uint4 x = reinterpret_cast<uint4 *>(a)[c];
        const uint4 y = __ldg(reinterpret_cast<const uint4 *>(b) + c);
        x.x -= y.x;
        x.y ^= y.y;
        x.z ^= y.z;
        x.w ^= y.w;
        reinterpret_cast<uint4 *>(a)[c] = x;
    }
}

extern "C" peel_status iblt_subtract(peel_iblt *a, const peel_iblt *b, void *stream) {
    if (!a || !b || a->C != b->C || a->r != b->r || a->seed != b->seed || a->subt != b->subt || a->blog != b->blog)
        return PEEL_EINVAL;
    a->insert_only = false;
    cudaStream_t s = (cudaStream_t)stream;
    prof_begin_call();
    {
        ProfScope ps("iblt_subtract", s);
        iblt_subtract_kernel<<<grid_for(a->C), 256, 0, s>>>((Cell *)(a->mem + a->L.cells),
                                                           (const Cell *)(b->mem + b->L.cells), a->C);
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}

// raw (writable) access: the table may no longer be insert-only
extern "C" void *iblt_cells(const peel_iblt *t) {
    if (!t) return nullptr;
    t->insert_only = false;
    return (void *)(t->mem + t->L.cells);
}

extern "C" peel_status iblt_to_hypergraph(const peel_iblt *t, const uint64_t *keys, uint64_t nkeys,
                                          uint32_t *edges, void *stream) {
    if (!t) return PEEL_EINVAL;
    if (nkeys == 0) return PEEL_OK;
    if (!keys || !edges) return PEEL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    prof_begin_call();
    unsigned g = grid_for(nkeys);
    {
        ProfScope ps("iblt_edges", s);
        switch (t->r) {
            case 2: iblt_edges_kernel<2><<<g, 256, 0, s>>>(t->C, t->seed_h, (const ull *)keys, nkeys, edges, t->subt, t->blog); break;
            case 3: iblt_edges_kernel<3><<<g, 256, 0, s>>>(t->C, t->seed_h, (const ull *)keys, nkeys, edges, t->subt, t->blog); break;
            case 4: iblt_edges_kernel<4><<<g, 256, 0, s>>>(t->C, t->seed_h, (const ull *)keys, nkeys, edges, t->subt, t->blog); break;
            case 5: iblt_edges_kernel<5><<<g, 256, 0, s>>>(t->C, t->seed_h, (const ull *)keys, nkeys, edges, t->subt, t->blog); break;
            case 6: iblt_edges_kernel<6><<<g, 256, 0, s>>>(t->C, t->seed_h, (const ull *)keys, nkeys, edges, t->subt, t->blog); break;
            case 7: iblt_edges_kernel<7><<<g, 256, 0, s>>>(t->C, t->seed_h, (const ull *)keys, nkeys, edges, t->subt, t->blog); break;
            case 8: iblt_edges_kernel<8><<<g, 256, 0, s>>>(t->C, t->seed_h, (const ull *)keys, nkeys, edges, t->subt, t->blog); break;
        }
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}

extern "C" void iblt_destroy(peel_iblt *t) { delete t; }
