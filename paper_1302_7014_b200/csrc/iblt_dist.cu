// iblt_dist.cu -- f3: one IBLT partitioned by cell range over P GPUs.
//
// Shard q owns cells [q cs, (q+1) cs) (cs = ceil(C/P) rounded up to 32).  Insert: every
// shard reads all keys and updates only its own cells (no communication).  Recovery runs the
// single-GPU round-synchronous schedule (iblt.cu) with the table split:
//   pure    each shard publishes its round-start pure cells as its slice of a C-bit bitmap
//           (one ncclAllGather per round; virtual shards share one bitmap)
//   find    for each local frontier entry (c, x): x is recovered by this entry iff c is the
//           lowest-index round-start-pure cell among h_1(x)..h_r(x) -- the owner rule, which
//           now reads other shards' pure bits from the gathered bitmap, so every key is found
//           exactly once.  The finder outputs x and sends it to every shard owning one of its
//           cells (itself included);
//   apply   each shard XOR-deletes every received key from its own cells of the key; a cell
//           whose count drops 2 -> 1 becomes a candidate;
//   retest  candidates still pure form the next local frontier.
// Same recovered set, rounds and per-round counts as the single-GPU table by construction
// (the owner rule and the round snapshot are identical); the tests check it against the oracle.
#include <nccl.h>
#include <stddef.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "iblt_common.cuh"

namespace peel {

static constexpr int IDB = 256;
static constexpr int IDQ = IDB;  // <= one push per thread per queue per iteration

struct IDCtl {
    ull fcnt[2];    // local frontier sizes by round parity
    ull ccnt;       // candidates this round
    ull nsend[8];   // per-destination message counts this round
    ull found;      // keys found by this shard this round
    uint32_t nonzero;
    uint32_t pad;
};
// the per-round reset clears ccnt .. found with one memset
static_assert(offsetof(IDCtl, found) == offsetof(IDCtl, ccnt) + 9 * sizeof(ull), "per-round counters contiguous");

static inline size_t ial(size_t x) { return (x + 255) & ~(size_t)255; }

static uint64_t id_cs(uint64_t C, int P) { return ((C + P - 1) / P + 31) & ~31ull; }

// common area (one per process): the C-bit pure bitmap (padded to P cs bits), the output
// counter, NCCL staging; then one region per local shard
struct IDLayout {
    size_t pure, outcnt, scratch, common;
    size_t ctl, cells, cand, F0, F1, clist, send, recv, shard;
};

static IDLayout id_layout(uint64_t C, int P) {
    const uint64_t cs = id_cs(C, P);
    IDLayout L;
    size_t o = 0;
    L.pure = o; o += ial(sizeof(uint32_t) * (P * cs / 32));
    L.outcnt = o; o += ial(sizeof(ull));
    L.scratch = o; o += ial(sizeof(ull) * (4 + 9 * 8));
    L.common = o;
    o = 0;
    L.ctl = o; o += ial(sizeof(IDCtl));
    L.cells = o; o += ial(sizeof(Cell) * cs);
    L.cand = o; o += ial(sizeof(uint32_t) * (cs / 32));
    L.F0 = o; o += ial(sizeof(ulonglong2) * cs);
    L.F1 = o; o += ial(sizeof(ulonglong2) * cs);
    L.clist = o; o += ial(sizeof(uint32_t) * cs);
    L.send = o; o += ial(sizeof(ull) * P * cs);   // a shard finds <= cs keys per round
    L.recv = o; o += ial(sizeof(ull) * P * cs);   // <= cs from each sender
    L.shard = o;
    return L;
}

struct IDArgs {
    Cell *cells;           // this shard's cells [c0, c1)
    uint32_t c0, ncl;      // first cell, cells owned
    uint32_t cs;           // cells per shard (the owner of cell c is c / cs)
    ull C, seed_h, seed_c;
    uint32_t blog;
    int P, p;
    uint32_t *pure;        // C-bit round-start pure bitmap (global cell ids)
    uint32_t *cand;        // local candidate bitmap
    uint32_t *clist;       // local candidate list (local ids)
    ulonglong2 *Fc, *Fn;   // frontier entries (global cell, key snapshot)
    const ull *pnF;        // this round's frontier size (device: no host round trip)
    ull *send;             // P segments of cs keys
    ull *out;              // recovered keys (output)
    ull *outcnt;
    ull cap_out;
    IDCtl *ctl;
    int par;               // parity of the next frontier
};

typedef BlockQueueT<ulonglong2, IDQ, IDB> IDEntQ;
typedef BlockQueueT<ull, IDQ, IDB> IDKeyQ;
typedef BlockQueueT<uint32_t, IDQ, IDB> IDCellQ;

template <int R>
__global__ void __launch_bounds__(IDB) idist_insert_kernel(IDArgs a, const ull *__restrict__ keys, ull nkeys) {
    for (ull i = blockIdx.x * (ull)IDB + threadIdx.x; i < nkeys; i += (ull)gridDim.x * IDB) {
        const ull x = __ldg(keys + i);
        uint32_t c[R];
        key_cells<R>(x, a.C, a.seed_h, false, c, a.blog);
        const uint32_t h = checksum(x, a.seed_c);
        #pragma unroll
        for (int j = 0; j < R; j++) {
            const uint32_t l = c[j] - a.c0;  // wraps for cells below c0
            if (l >= a.ncl) continue;
            Cell *p = a.cells + l;
            atomicAdd(&p->count, 1u);
            atomicXor(&p->keySum, x);
            atomicXor(&p->hashSum, h);
        }
    }
}

// pure (R28): count 1, matching checksum, and c (global id) is one of the key's cells
template <int R>
__device__ __forceinline__ bool id_pure(const Cell &v, uint32_t c, const IDArgs &a) {
    return is_pure(v, a.seed_c) && cell_of_key<R>(c, v.keySum, a.C, a.seed_h, false, a.blog);
}

// round 1: the shard's pure cells -> frontier entries and pure bits
template <int R>
__global__ void __launch_bounds__(IDB) idist_scan_kernel(IDArgs a) {
    __shared__ IDEntQ q;
    bq_init(q);
    __syncthreads();
    ull *cnt = &a.ctl->fcnt[a.par];
    int slot = 0;
    for (ull base = (ull)blockIdx.x * IDB; base < a.ncl; base += (ull)gridDim.x * IDB) {
        const ull l = base + threadIdx.x;
        if (l < a.ncl) {
            const Cell v = ld_cell_cg(a.cells + l);
            if (id_pure<R>(v, a.c0 + (uint32_t)l, a)) {
                const uint32_t c = a.c0 + (uint32_t)l;
                bq_push(q, slot, make_ulonglong2(c, v.keySum), a.Fn, cnt);
                atomicOr(a.pure + (c >> 5), 1u << (c & 31));
            }
        }
        bq_flush(q, slot, a.Fn, cnt);
        slot ^= 1;
    }
}

// find: the owner rule over the gathered pure bitmap; the finder outputs the key and sends
// it to every shard owning one of its cells
template <int R>
__global__ void __launch_bounds__(IDB) idist_find_kernel(IDArgs a) {
    __shared__ IDKeyQ qo;
    __shared__ IDKeyQ qs[8];
    bq_init(qo);
    for (int d = 0; d < 8; d++) bq_init(qs[d]);
    __syncthreads();
    ull found = 0;
    int slot = 0;
    const ull nF = ld_cg_u64(a.pnF);
    for (ull base = (ull)blockIdx.x * IDB; base < nF; base += (ull)gridDim.x * IDB) {
        const ull i = base + threadIdx.x;
        uint32_t dmask = 0;
        ull x = 0;
        if (i < nF) {
            const ulonglong2 ent = __ldcg(a.Fc + i);
            const uint32_t c = (uint32_t)ent.x;
            x = ent.y;
            uint32_t h[R];
            key_cells<R>(x, a.C, a.seed_h, false, h, a.blog);
            uint32_t pw[R];
            #pragma unroll
            for (int j = 0; j < R; j++) pw[j] = ld_cg_u32(a.pure + (h[j] >> 5));
            bool owner = false, done = false;
            #pragma unroll
            for (int j = 0; j < R; j++) {
                if (!done && h[j] == c) { done = true; owner = true; }
                if (!done && (pw[j] >> (h[j] & 31) & 1u)) done = true;
            }
            if (owner) {
                found++;
                bq_push(qo, slot, x, a.out, a.outcnt);
                #pragma unroll
                for (int j = 0; j < R; j++) dmask |= 1u << (h[j] / a.cs);
            }
        }
        // one push per destination; d is warp-uniform (each coalesced group targets one queue)
        for (int d = 0; d < a.P; d++)
            if (dmask >> d & 1u) bq_push(qs[d], slot, x, a.send + (ull)d * a.cs, &a.ctl->nsend[d]);
        bq_flush(qo, slot, a.out, a.outcnt, a.cap_out);
        for (int d = 0; d < a.P; d++) bq_flush(qs[d], slot, a.send + (ull)d * a.cs, &a.ctl->nsend[d]);
        slot ^= 1;
    }
    block_add<IDB>(&a.ctl->found, found);
}

// apply: XOR-delete every received key from this shard's cells; 2 -> 1 drops are candidates
template <int R>
__global__ void __launch_bounds__(IDB) idist_apply_kernel(IDArgs a, const ull *__restrict__ recv, ull nrecv) {
    __shared__ IDCellQ qc;
    bq_init(qc);
    __syncthreads();
    int slot = 0;
    for (ull base = (ull)blockIdx.x * IDB; base < nrecv; base += (ull)gridDim.x * IDB) {
        const ull i = base + threadIdx.x;
        if (i < nrecv) {
            const ull x = __ldcg(recv + i);
            uint32_t h[R];
            key_cells<R>(x, a.C, a.seed_h, false, h, a.blog);
            const uint32_t hx = checksum(x, a.seed_c);
            uint32_t now[R];
            #pragma unroll
            for (int j = 0; j < R; j++) {
                const uint32_t l = h[j] - a.c0;
                now[j] = 0;
                if (l < a.ncl) {
                    Cell *p = a.cells + l;
                    now[j] = atomicAdd(&p->count, 0xFFFFFFFFu) - 1u;
                    atomicXor(&p->keySum, x);
                    atomicXor(&p->hashSum, hx);
                }
            }
            #pragma unroll
            for (int j = 0; j < R; j++) {
                const uint32_t l = h[j] - a.c0;
                if (l < a.ncl && now[j] == 1u) {
                    const uint32_t bit = 1u << (l & 31);
                    if (!(atomicOr(a.cand + (l >> 5), bit) & bit)) bq_push(qc, slot, l, a.clist, &a.ctl->ccnt);
                }
            }
        }
        bq_flush(qc, slot, a.clist, &a.ctl->ccnt);
        slot ^= 1;
    }
}

// retire this round's pure bits of the shard
__global__ void __launch_bounds__(IDB) idist_clear_kernel(IDArgs a) {
    const ull nF = ld_cg_u64(a.pnF);
    for (ull i = blockIdx.x * (ull)IDB + threadIdx.x; i < nF; i += (ull)gridDim.x * IDB) {
        const uint32_t c = (uint32_t)__ldcg(&a.Fc[i].x);
        atomicAnd(a.pure + (c >> 5), ~(1u << (c & 31)));
    }
}

// retest: candidates still pure -> the next local frontier and pure bits
template <int R>
__global__ void __launch_bounds__(IDB) idist_retest_kernel(IDArgs a) {
    __shared__ IDEntQ q;
    bq_init(q);
    __syncthreads();
    const ull ncand = ld_cg_u64(&a.ctl->ccnt);
    ull *cnt = &a.ctl->fcnt[a.par];
    int slot = 0;
    for (ull base = (ull)blockIdx.x * IDB; base < ncand; base += (ull)gridDim.x * IDB) {
        const ull i = base + threadIdx.x;
        if (i < ncand) {
            const uint32_t l = __ldcg(a.clist + i);
            atomicAnd(a.cand + (l >> 5), ~(1u << (l & 31)));
            const Cell v = ld_cell_cg(a.cells + l);
            if (id_pure<R>(v, a.c0 + l, a)) {
                const uint32_t c = a.c0 + l;
                bq_push(q, slot, make_ulonglong2(c, v.keySum), a.Fn, cnt);
                atomicOr(a.pure + (c >> 5), 1u << (c & 31));
            }
        }
        bq_flush(q, slot, a.Fn, cnt);
        slot ^= 1;
    }
}

__global__ void __launch_bounds__(IDB) idist_nonzero_kernel(IDArgs a) {
    uint32_t nz = 0;
    for (ull l = blockIdx.x * (ull)IDB + threadIdx.x; l < a.ncl; l += (ull)gridDim.x * IDB) {
        const Cell v = ld_cell_cg(a.cells + l);
        nz |= (v.count | v.hashSum) != 0u || v.keySum != 0ull;
    }
    if (__any_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) atomicOr(&a.ctl->nonzero, 1u);
}

static unsigned idgrid(ull work) {
    ull b = (work + IDB - 1) / IDB, cap = (ull)num_sms() * 8;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

static ull id_mix64(ull z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct IDShard {
    int q;
    uint32_t c0, ncl;
    char *base;
    IDCtl *ctl;
};

template <int R>
static peel_status run_iblt_dist(peel_comm *c, uint64_t C, uint64_t seed, uint32_t blog, const uint64_t *keys,
                                 uint64_t nkeys, const Cell *cells_in, uint64_t *out_keys, uint64_t cap_keys,
                                 uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round, uint32_t cap,
                                 int *complete, char *mem, cudaStream_t s) {
    const int P = c->P;
    const uint64_t cs = id_cs(C, P);
    const IDLayout L = id_layout(C, P);
    const ull G = 0x9E3779B97F4A7C15ull;
    uint32_t *pure = (uint32_t *)(mem + L.pure);
    ull *outcnt = (ull *)(mem + L.outcnt);
    ull *dsum = (ull *)(mem + L.scratch);
    std::vector<IDShard> sh;
    for (int q = 0; q < P; q++) {
        if (!c->virt && q != c->rank) continue;
        IDShard d;
        d.q = q;
        d.c0 = (uint32_t)std::min<uint64_t>(C, (uint64_t)q * cs);
        d.ncl = (uint32_t)(std::min<uint64_t>(C, (uint64_t)(q + 1) * cs) - d.c0);
        d.base = mem + L.common + (c->virt ? (size_t)q * L.shard : 0);
        d.ctl = (IDCtl *)(d.base + L.ctl);
        sh.push_back(d);
    }
    auto args = [&](const IDShard &d, int cur) {
        IDArgs a;
        memset(&a, 0, sizeof a);
        a.cells = (Cell *)(d.base + L.cells);
        a.c0 = d.c0;
        a.ncl = d.ncl;
        a.cs = (uint32_t)cs;
        a.C = C;
        a.seed_h = id_mix64((seed ^ 0x6A09E667F3BCC909ull) + G);
        a.seed_c = id_mix64((seed ^ 0xBB67AE8584CAA73Bull) + G);
        a.blog = blog;
        a.P = P;
        a.p = d.q;
        a.pure = pure;
        a.cand = (uint32_t *)(d.base + L.cand);
        a.clist = (uint32_t *)(d.base + L.clist);
        ulonglong2 *F[2] = {(ulonglong2 *)(d.base + L.F0), (ulonglong2 *)(d.base + L.F1)};
        a.Fc = F[cur];
        a.Fn = F[cur ^ 1];
        a.pnF = &d.ctl->fcnt[cur];
        a.send = (ull *)(d.base + L.send);
        a.out = (ull *)out_keys;
        a.outcnt = outcnt;
        a.cap_out = cap_keys;
        a.ctl = d.ctl;
        a.par = cur ^ 1;
        return a;
    };
    // error protocol as dist.cu's (peel.h "Errors"): local failures are carried in the
    // failure words of the collectives, every rank leaves at the same one
    peel_status lst = PEEL_OK;
    auto cu = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess && lst == PEEL_OK) {
            set_cuda_error(e, what);
            lst = PEEL_ECUDA;
        }
        return lst == PEEL_OK;
    };
    // zero the common area and every local shard's control block, cells and candidate bits
    cu(cudaMemsetAsync(mem, 0, L.common, s), "memset");
    for (auto &d : sh) {
        if (!cu(cudaMemsetAsync(d.base, 0, L.F0, s), "memset")) break;  // ctl, cells, cand
        IDArgs a = args(d, 1);                                          // round 1's frontier goes to F[0]
        if (cells_in) {
            if (!cu(cudaMemcpyAsync(a.cells, cells_in + d.c0, sizeof(Cell) * d.ncl, cudaMemcpyDeviceToDevice, s), "cells_in"))
                break;
        } else if (nkeys) {
            ProfScope ps("iblt_dist_insert", s);
            idist_insert_kernel<R><<<idgrid(nkeys), IDB, 0, s>>>(a, (const ull *)keys, nkeys);
        }
        ProfScope ps("iblt_dist_scan", s);
        idist_scan_kernel<R><<<idgrid(d.ncl), IDB, 0, s>>>(a);
    }
    cu(cudaGetLastError(), "build launch");
    if (lst != PEEL_OK && c->virt) return lst;

    std::vector<IDCtl> hc(sh.size());
    auto fetch = [&]() {
        if (!c->virt && !c->host) {  // after NCCL work: the watchdog sync, before the copies
            const peel_status ws = comm_sync(c, s);  // (pageable copies would block out of its sight)
            if (ws != PEEL_OK && lst == PEEL_OK) lst = ws;
            if (lst != PEEL_OK) return;
        }
        for (size_t i = 0; i < sh.size(); i++)
            cu(cudaMemcpyAsync(&hc[i], sh[i].ctl, sizeof(IDCtl), cudaMemcpyDeviceToHost, s), "fetch");
        cu(cudaStreamSynchronize(s), "fetch");
    };
    // global sums over shards / ranks of (v0, v1) and the failure word: out[2] = failed ranks
    auto gsum = [&](ull v0, ull v1, ull out[3]) -> peel_status {
        out[0] = v0;
        out[1] = v1;
        out[2] = lst != PEEL_OK ? 1 : 0;
        if (c->virt) return PEEL_OK;
        return comm_allreduce_sum(c, out, 3, dsum, s);
    };
    auto leave = [&](bool peer_failed) -> peel_status {
        if (lst != PEEL_OK) return lst;
        return peer_failed ? PEEL_EPEER : PEEL_OK;
    };
    fetch();
    if (lst != PEEL_OK && c->virt) return lst;
    ull g[3];
    {
        ull f = 0;
        for (auto &h : hc) f += h.fcnt[0];
        peel_status st = gsum(f, 0, g);
        if (st != PEEL_OK) return st;
        if (g[2]) return leave(true);
    }
    uint32_t t = 0;
    std::vector<ull> cnt_mat((size_t)P * P), rows((size_t)P * (P + 1));
    bool trunc = false;
    while (g[0] > 0) {
        if (t == 65536u) {  // round limit, as iblt_peel's (R28: forged signed tables can cycle)
            trunc = true;
            break;
        }
        t++;
        const int cur = (t - 1) & 1;  // round t's frontier: F[(t-1) & 1]
        if (comm_fault(c, t) && lst == PEEL_OK) {
            set_cuda_error(cudaErrorUnknown, "PEEL_FAULT injected failure");
            lst = PEEL_ECUDA;
        }
        for (auto &d : sh) {
            cu(cudaMemsetAsync(&d.ctl->fcnt[cur ^ 1], 0, sizeof(ull), s), "memset");
            cu(cudaMemsetAsync(&d.ctl->ccnt, 0, sizeof(ull) * 10, s), "memset");  // ccnt, nsend[8], found
        }
        // pure bits of every shard (ranks: in-place allgather of the slices)
        if (!c->virt) {
            peel_status sg = comm_allgather_dev(c, pure + (size_t)c->rank * (cs / 32), pure, cs / 32 * sizeof(uint32_t), s);
            if (sg != PEEL_OK) return sg;
        }
        // find (frontier sizes are read on the device: hc[] still holds them from the end of
        // the previous round, which sizes the grids)
        for (size_t i = 0; i < sh.size() && lst == PEEL_OK; i++) {
            IDArgs a = args(sh[i], cur);
            const ull nF = hc[i].fcnt[cur];
            if (!nF) continue;
            ProfScope ps("iblt_dist_find", s);
            idist_find_kernel<R><<<idgrid(nF), IDB, 0, s>>>(a);
        }
        cu(cudaGetLastError(), "find launch");
        fetch();
        if (lst != PEEL_OK && c->virt) return lst;
        // exchange (self-delivery included): cnt_mat[src * P + dst]; every rank's row carries
        // its failure word
        if (c->virt) {
            for (int q = 0; q < P; q++)
                for (int d = 0; d < P; d++) cnt_mat[(size_t)q * P + d] = hc[q].nsend[d];
        } else {
            std::vector<ull> mine(P + 1, 0);
            for (int d = 0; d < P; d++) mine[d] = hc[0].nsend[d];
            mine[P] = lst != PEEL_OK ? 1 : 0;
            peel_status sg = comm_allgather_u64(c, mine.data(), rows.data(), P + 1, dsum + 4, s);
            if (sg != PEEL_OK) return lst != PEEL_OK ? lst : sg;
            bool peer_failed = false;
            for (int q = 0; q < P; q++) peer_failed |= rows[(size_t)q * (P + 1) + P] != 0;
            if (lst != PEEL_OK || peer_failed) return leave(peer_failed);
            for (int q = 0; q < P; q++)
                for (int d = 0; d < P; d++) cnt_mat[(size_t)q * P + d] = rows[(size_t)q * (P + 1) + d];
        }
        // capacity of every receiver, from the gathered matrix (all ranks agree)
        for (int dst = 0; dst < P; dst++)
            for (int src = 0; src < P; src++)
                if (cnt_mat[(size_t)src * P + dst] > cs) return PEEL_ENOMEM;
        std::vector<ull> nrecv(sh.size(), 0);
        for (size_t i = 0; i < sh.size(); i++) {
            const int dst = sh[i].q;
            ull *recv = (ull *)(sh[i].base + L.recv);
            // self-delivery (and every delivery between virtual shards) is a device copy, packed
            // first; the other ranks' keys follow in increasing source rank
            ull off = 0;
            for (int src = 0; src < P; src++) {
                if (!(c->virt || src == dst)) continue;
                const ull cn = cnt_mat[(size_t)src * P + dst];
                if (!cn) continue;
                const char *sb = mem + L.common + (c->virt ? (size_t)src * L.shard : 0) + L.send;
                cu(cudaMemcpyAsync(recv + off, (const ull *)sb + (size_t)dst * cs, sizeof(ull) * cn,
                                   cudaMemcpyDeviceToDevice, s), "self delivery");
                off += cn;
            }
            if (!c->virt) {
                std::vector<const char *> sp(P);
                std::vector<ull> sbytes(P), rbytes(P);
                const ull *sb = (const ull *)(sh[i].base + L.send);
                for (int q = 0; q < P; q++) {
                    sp[q] = (const char *)(sb + (size_t)q * cs);
                    sbytes[q] = q == dst ? 0 : sizeof(ull) * cnt_mat[(size_t)dst * P + q];
                    rbytes[q] = q == dst ? 0 : sizeof(ull) * cnt_mat[(size_t)q * P + dst];
                }
                peel_status sx = comm_alltoallv(c, sp.data(), sbytes.data(), (char *)(recv + off), rbytes.data(), s);
                if (sx != PEEL_OK) return sx;
                for (int q = 0; q < P; q++) off += rbytes[q] / sizeof(ull);
            }
            nrecv[i] = off;
        }
        // apply, retire the round's pure bits, retest the candidates
        ull found = 0;
        for (auto &h : hc) found += h.found;
        for (size_t i = 0; i < sh.size() && lst == PEEL_OK; i++) {
            IDArgs a = args(sh[i], cur);
            if (nrecv[i]) {
                ProfScope ps("iblt_dist_apply", s);
                idist_apply_kernel<R><<<idgrid(nrecv[i]), IDB, 0, s>>>(a, (const ull *)(sh[i].base + L.recv), nrecv[i]);
            }
        }
        ull nf = 0;
        for (size_t i = 0; i < sh.size() && lst == PEEL_OK; i++) {
            IDArgs a = args(sh[i], cur);
            const ull nF = hc[i].fcnt[cur];
            ProfScope ps("iblt_dist_retest", s);
            if (nF) idist_clear_kernel<<<idgrid(nF), IDB, 0, s>>>(a);
            // candidates <= keys received x r (sized from the host's receive count)
            idist_retest_kernel<R><<<idgrid(std::min<ull>(nrecv[i] * R, sh[i].ncl)), IDB, 0, s>>>(a);
        }
        cu(cudaGetLastError(), "apply launch");
        fetch();
        if (lst != PEEL_OK && c->virt) return lst;
        for (auto &h : hc) nf += h.fcnt[cur ^ 1];
        peel_status st = gsum(nf, found, g);
        if (st != PEEL_OK) return st;
        if (g[2]) return leave(true);
        if (t <= cap && per_round) per_round[t - 1] = g[1];
    }
    // completeness: every cell of every shard zero
    for (auto &d : sh) {
        IDArgs a = args(d, 0);
        ProfScope ps("iblt_dist_nonzero", s);
        idist_nonzero_kernel<<<idgrid(d.ncl), IDB, 0, s>>>(a);
    }
    cu(cudaGetLastError(), "nonzero launch");
    fetch();
    ull nz = 0, nout = 0;
    for (auto &h : hc) nz |= h.nonzero;
    cu(cudaMemcpyAsync(&nout, outcnt, sizeof(ull), cudaMemcpyDeviceToHost, s), "outcnt");
    cu(cudaStreamSynchronize(s), "sync");
    prof_collect();
    if (lst != PEEL_OK && c->virt) return lst;
    peel_status st = gsum(nz ? 1 : 0, 0, g);
    if (st != PEEL_OK) return st;
    if (g[2]) return leave(true);
    *rounds = t;
    *nrecovered = nout;
    if (complete) *complete = g[0] ? 0 : 1;
    if (nout > cap_keys || t > cap || trunc) return PEEL_ETRUNC;
    return PEEL_OK;
}

}  // namespace peel

using namespace peel;

extern "C" size_t iblt_dist_mem_bytes(const peel_comm *c, uint64_t cells, uint32_t r) {
    if (!c || r < 2 || r > 8 || cells < r || cells >= (1ull << 32) || c->P < 1 || c->P > 8) return 0;
    const IDLayout L = id_layout(cells, c->P);
    return L.common + (c->virt ? (size_t)c->P : 1) * L.shard;
}

static peel_status idist_entry(peel_comm *c, uint64_t cells, uint32_t r, uint64_t seed, uint32_t flags,
                               const uint64_t *keys, uint64_t nkeys, const void *cells_in, uint64_t *out_keys,
                               uint64_t cap_keys, uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round,
                               uint32_t cap, int *complete, void *mem, size_t mem_bytes, void *stream) {
    if (!c) return PEEL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t need = iblt_dist_mem_bytes(c, cells, r);
    peel_status v = PEEL_OK;
    uint32_t blog = 0;
    if (!need || !nrecovered || !rounds || !mem || (nkeys && !keys) || (cap_keys && !out_keys)) v = PEEL_EINVAL;
    else if (cells_in && ((uintptr_t)cells_in & 15)) v = PEEL_EINVAL;
    else if (flags & ~(IBLT_FLAG_BLOCKED | (0xFFu << IBLT_BLOCK_LOG_SHIFT))) v = PEEL_EINVAL;  // no subtables / signed
    else if (flags & IBLT_FLAG_BLOCKED) {
        blog = IBLT_BLOCK_LOG(flags) ? IBLT_BLOCK_LOG(flags) : 16u;
        if (blog < 4 || blog > 30 || cells % (1ull << blog) || (1ull << blog) < r) v = PEEL_EINVAL;
    }
    if (v == PEEL_OK && mem_bytes < need) v = PEEL_ENOMEM;
    v = comm_agree(c, v, s);  // every rank leaves together if any rank rejects its arguments
    if (v != PEEL_OK) return v;
    prof_begin_call();
    char *m = (char *)mem;
    const Cell *ci = (const Cell *)cells_in;
    switch (r) {
        case 2: return run_iblt_dist<2>(c, cells, seed, blog, keys, nkeys, ci, out_keys, cap_keys, nrecovered, rounds, per_round, cap, complete, m, s);
        case 3: return run_iblt_dist<3>(c, cells, seed, blog, keys, nkeys, ci, out_keys, cap_keys, nrecovered, rounds, per_round, cap, complete, m, s);
        case 4: return run_iblt_dist<4>(c, cells, seed, blog, keys, nkeys, ci, out_keys, cap_keys, nrecovered, rounds, per_round, cap, complete, m, s);
        case 5: return run_iblt_dist<5>(c, cells, seed, blog, keys, nkeys, ci, out_keys, cap_keys, nrecovered, rounds, per_round, cap, complete, m, s);
        case 6: return run_iblt_dist<6>(c, cells, seed, blog, keys, nkeys, ci, out_keys, cap_keys, nrecovered, rounds, per_round, cap, complete, m, s);
        case 7: return run_iblt_dist<7>(c, cells, seed, blog, keys, nkeys, ci, out_keys, cap_keys, nrecovered, rounds, per_round, cap, complete, m, s);
        case 8: return run_iblt_dist<8>(c, cells, seed, blog, keys, nkeys, ci, out_keys, cap_keys, nrecovered, rounds, per_round, cap, complete, m, s);
    }
    return PEEL_EINVAL;
}

extern "C" peel_status iblt_dist_recover(peel_comm *c, uint64_t cells, uint32_t r, uint64_t seed, uint32_t flags,
                                         const uint64_t *keys, uint64_t nkeys, uint64_t *out_keys, uint64_t cap_keys,
                                         uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round, uint32_t cap,
                                         int *complete, void *mem, size_t mem_bytes, void *stream) {
    return idist_entry(c, cells, r, seed, flags, keys, nkeys, nullptr, out_keys, cap_keys, nrecovered, rounds,
                       per_round, cap, complete, mem, mem_bytes, stream);
}

extern "C" peel_status iblt_dist_recover_cells(peel_comm *c, const void *cells_in, uint64_t cells, uint32_t r,
                                               uint64_t seed, uint32_t flags, uint64_t *out_keys, uint64_t cap_keys,
                                               uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round,
                                               uint32_t cap, int *complete, void *mem, size_t mem_bytes,
                                               void *stream) {
    return idist_entry(c, cells, r, seed, flags, nullptr, 0, cells_in, out_keys, cap_keys, nrecovered, rounds,
                       per_round, cap, complete, mem, mem_bytes, stream);
}
