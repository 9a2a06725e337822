/*
 * peel.h -- C-ABI of libpeel.so: round-synchronous parallel peeling of random
 * r-uniform hypergraphs to the k-core, and IBLT recovery, on NVIDIA B200
 * (sm_100a).  Plain pointers and sizes only; no torch or CUDA types.
 *
 * Citations: "P:n" = line n of the paper (Jiang, Mitzenmacher, Thaler,
 * "Parallel Peeling Algorithms", arXiv 1302.7014, PAPER.md); "S:n" = SPEC.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - "dev" pointers are CUDA device pointers (e.g. torch tensor data_ptr());
 *   "host" pointers are ordinary CPU memory.  The caller owns every buffer it
 *   passes; the library never frees them.
 * - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   Everything is stream-ordered on it.  Calls that return host scalars
 *   (peel_kcore, iblt_peel, ...) synchronise `stream` before returning.
 * - Errors are returned as peel_status; nothing is thrown or aborted across
 *   the ABI.  Arguments are validated before any launch (PEEL_EINVAL).
 *   Outputs are meaningful only on PEEL_OK (and on PEEL_ETRUNC, see below).
 * - Vertex ids are u32 (n <= 2^32); edge ids are u32 (m < 2^32); 2 <= r <= 8.
 * - Not thread-safe per stream: concurrent calls must use distinct streams and
 *   workspaces.
 */
#ifndef PEEL_H_
#define PEEL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PEEL_OK = 0,
    PEEL_EINVAL = 1,    /* bad argument, or an input edge with a vertex id >= n or a repeated vertex */
    PEEL_ENOMEM = 2,    /* workspace too small / allocation failed */
    PEEL_ECUDA = 3,     /* a CUDA runtime error (peel_last_cuda_error() has the text) */
    PEEL_ETRUNC = 4,    /* more rounds than the caller's `cap`; rounds and the first cap entries are valid */
    PEEL_ENCCL = 5,     /* an NCCL error (multi-GPU entry points) */
    PEEL_EOVERFLOW = 6, /* packed k<=2 state cannot hold this degree x edge-id range (see peel_kcore) */
    PEEL_EPEER = 7      /* multi-rank calls: another rank of the communicator failed; every rank
                           leaves the call at the same collective (the failing rank returns its
                           own status) */
} peel_status;

/* Human-readable name of a status code (static storage). */
const char *peel_strerror(int status);
/* Text of the last CUDA error seen by this process's library calls (static storage). */
const char *peel_last_cuda_error(void);
/* ABI version of this header (bumped on any signature change). */
int peel_abi_version(void);
#define PEEL_ABI_VERSION 2

/* ======================================================================= */
/* a1 -- generator: G^r_{n,cn} and IBLT keys (counter-based) */
/* ======================================================================= */

/*
 * peel_gen_hypergraph -- fill edges[m][r] (dev, u32, row-major) with m
 * independent hyperedges of r DISTINCT vertices chosen uniformly from [0,n)
 * ("cn hyperedges, where each hyperedge consists of r distinct
 * vertices"; "each edge is chosen independently and uniformly").
 * Edge e is a pure function of (seed, n, r, e): draw j is half j%2 of
 * Philox4x32-10(ctr = {e_lo, e_hi, j/2, 'EDGE'}, key = {seed_lo, seed_hi}),
 * mapped to vertex umulhi64(draw, n), rejected if already in the edge.
 * Vertex order within an edge is draw order.  Duplicate edges may occur
 * (hashing model).
 * EINVAL: r < 2, r > 8, n < r, n > 2^32, m >= 2^32, edges == NULL with m > 0.
 */
peel_status peel_gen_hypergraph(uint64_t n, uint64_t m, uint32_t r, uint64_t seed,
                                uint32_t *edges, void *stream);

/*
 * peel_gen_partitioned -- the subtable model: r | n, vertex class
 * c = [c n/r, (c+1) n/r), and edge e has exactly one vertex per class: the
 * class-c vertex is c n/r + umulhi64(draw c, n/r), draw c = half c%2 of
 * Philox4x32-10(ctr = {e_lo, e_hi, c/2, 'SUBT'}, key = {seed_lo, seed_hi}).
 * EINVAL: r < 2, r > 8, n % r != 0, n > 2^32, m >= 2^32.
 */
peel_status peel_gen_partitioned(uint64_t n, uint64_t m, uint32_t r, uint64_t seed, uint32_t *edges, void *stream);

/*
 * peel_gen_keys -- keys[i] (dev, u64) = i-th output of a SplitMix64 stream
 * with state `seed`: mix64(seed + (i+1) * 0x9E3779B97F4A7C15).  A bijection of
 * i, so the nkeys keys are distinct (the IBLT stores a set).
 */
peel_status peel_gen_keys(uint64_t nkeys, uint64_t seed, uint64_t *keys, void *stream);

/* ======================================================================= */
/* a2-a7 -- k-core by round-synchronous parallel peeling                    */
/* ======================================================================= */

/* flags */
#define PEEL_FLAG_CSR 1u /* force the general-k incidence (CSR) path even for k <= 2 */
/* The subround (subtable) variant of P:565-579: vertices in r classes
 * [c n/r, (c+1) n/r) (r must divide n; k <= 2); round i = r subrounds, subround j
 * removing the class-j vertices of degree < k at ITS start, after subrounds
 * 1..j-1 applied.  With this flag `rounds` is the flattened index (i-1) r + j of
 * the last subround that removed a vertex (Table 4's "subrounds"), and
 * survivors / killed / peel_round are per flattened subround (Table 5). */
#define PEEL_FLAG_SUBROUNDS 2u

/*
 * Bytes of device workspace peel_kcore needs for (n, m, r, k, flags).
 * Returns 0 if the arguments are invalid.
 */
size_t peel_kcore_workspace_bytes(uint64_t n, uint64_t m, uint32_t r, uint32_t k, uint32_t flags);

/*
 * peel_kcore -- round-synchronous parallel peeling to the k-core
 * ("in each round, all vertices of degree less than k and their
 * adjacent edges are removed in parallel"; an edge is peeled when
 * an adjacent vertex is; the k-core is the maximal sub-hypergraph with all
 * degrees >= k).
 *
 * Round t removes F_t = {alive v : deg_t(v) < k}, deg_t the number of alive
 * edges at the START of round t (a snapshot; degree-0 vertices included),
 * then every alive edge with an endpoint in F_t.  The loop stops at the first
 * round with F_t empty; that terminal round is not counted.
 *
 * in:  edges     dev u32 [m][r], row-major, read-only.  Every id < n and the
 *                r ids of an edge distinct, else PEEL_EINVAL (checked on device).
 *                Edges are a multiset (duplicates allowed).
 *      n, m, r, k  sizes; k = 0 peels nothing (rounds = 0).
 *      flags     0, PEEL_FLAG_CSR or PEEL_FLAG_SUBROUNDS.
 * out: core_mask dev u8 [n]: 1 iff v is in the k-core.
 *      rounds    host u32: number of rounds with F_t non-empty.
 *      survivors host u64 [cap] (nullable): survivors[t-1] = |alive vertices|
 *                after round t, t = 1..min(rounds, cap).
 *      killed    host u64 [cap] (nullable): edges removed in round t.
 *      peel_round dev u32 [n] (nullable): round in which v was removed, 0 if
 *                v is in the core (a schedule certificate for tests).
 * workspace: dev, >= peel_kcore_workspace_bytes(n, m, r, k, flags) bytes,
 *      any contents; clobbered.
 * Blocking: synchronises `stream` before returning.
 * Status: PEEL_ETRUNC if rounds > cap (or > 65536): rounds is exact, the
 *      first cap entries are written.  (PEEL_EOVERFLOW is reserved: the k <= 2
 *      packed state -- count in the low 32 bits, edge-id sum mod 2^32 above it --
 *      cannot overflow for m < 2^32.)
 */
peel_status peel_kcore(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r, uint32_t k,
                       uint32_t flags, uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors,
                       uint64_t *killed, uint32_t cap, uint32_t *peel_round, void *workspace,
                       size_t ws_bytes, void *stream);

/*
 * peel_kcore_host -- the same computation with HOST input and output:
 * edges_host u32 [m][r] and core_mask_host u8 [n] are CPU memory (pinned for
 * full copy speed); the host->device copy of the edges and the device->host
 * copy of the mask are part of the call.  For n > 2^23 (k <= 2) the edges are
 * copied in 16 chunks that the build partitions as they land, and the mask
 * comes back as 64 chunks of which only those holding a core vertex are copied;
 * host threads zero the rest of core_mask_host during the peel (its previous
 * contents are irrelevant either way).  workspace must hold
 * peel_kcore_host_workspace_bytes(n, m, r, k, flags) bytes of device memory.
 */
size_t peel_kcore_host_workspace_bytes(uint64_t n, uint64_t m, uint32_t r, uint32_t k, uint32_t flags);
peel_status peel_kcore_host(const uint32_t *edges_host, uint64_t n, uint64_t m, uint32_t r,
                            uint32_t k, uint32_t flags, uint8_t *core_mask_host, uint32_t *rounds,
                            uint64_t *survivors, uint64_t *killed, uint32_t cap, void *workspace,
                            size_t ws_bytes, void *stream);

/* ======================================================================= */
/* e1 -- independent-trial sweeps (the paper's simulation protocol)  */
/* ======================================================================= */

/*
 * peel_sweep -- for each trial t in [0, ntrials): generate G^r_{n, m[t]} with
 * seed seeds[t] (exactly peel_gen_hypergraph(n, m[t], r, seeds[t])) and peel it
 * to its k-core (exactly peel_kcore); report out_rounds[t] (host u32) and
 * out_core[t] (host u64: k-core vertices; "Failed" in Table 1 iff > 0).
 * m[], seeds[] are host arrays.  For k = 2, r <= 4 and n <= 2^22 each trial is peeled by
 * a group of co-resident CTAs with 32-bit L2-resident states and edge rows regenerated
 * from (seeds[t], e) (PEEL_SWEEP_GROUPS=0 turns it off); a trial whose
 * 32-bit count field would overflow is redone on the union path.  Otherwise trials are
 * processed `batch` at a time as one disjoint-union hypergraph (the synchronous peel of a
 * disjoint union is the trials' synchronous peels in lockstep).  Either way
 * 1 <= batch <= 1024, batch * n <= 2^32 and batch * max(m) < 2^32.  Multi-GPU sweeps shard the trial index range across
 * ranks (no data-path collective); see paper_1302_7014_b200/trials.py.
 * workspace: dev, peel_sweep_workspace_bytes(n, max(m), r, k, batch) bytes.
 * Blocking (one stream sync per batch).
 */
size_t peel_sweep_workspace_bytes(uint64_t n, uint64_t max_m, uint32_t r, uint32_t k, uint32_t batch);
peel_status peel_sweep(uint64_t n, uint32_t r, uint32_t k, const uint64_t *m, const uint64_t *seeds,
                       uint64_t ntrials, uint32_t batch, uint32_t *out_rounds, uint64_t *out_core,
                       void *workspace, size_t ws_bytes, void *stream);

/* ======================================================================= */
/* e2 -- one instance partitioned by vertex range over P GPUs               */
/* ======================================================================= */

/*
 * Rank p of P owns vertices [p n / P, (p+1) n / P).  The edge list is
 * replicated (read-only) on every rank.  Each round: local kills, ONE
 * all-to-all of killed edge ids to the other owners of their endpoints (NCCL
 * grouped send/recv), receiver-side exactly-once application, and a 3-word
 * allreduce (|F_{t+1}|, edges killed, errors) that is the termination test.
 * Results are bit-identical to peel_kcore (k <= 2; EINVAL for k >= 3).
 *
 * peel_comm_unique_id: fill 128 bytes with an NCCL unique id (rank 0), to be
 *   broadcast to the other ranks by the caller (e.g. torch.distributed).
 * peel_comm_init: NCCL communicator, one process per GPU (current device).
 * peel_comm_init_virtual: P shards inside ONE process on ONE GPU, the
 *   all-to-all done by device copies through the same send/receive buffers
 *   and kernels -- the partitioning logic testable without P GPUs.
 * peel_comm_init_host: a rank communicator whose collectives go through three
 *   caller-supplied HOST callbacks (every rank one process; e.g. torch.distributed
 *   gloo), with device<->host staging inside the library.  It runs exactly the
 *   per-rank protocol of the NCCL communicator (count exchange, per-peer payload,
 *   allreduce, error word) and needs no GPU per rank: no kernel waits on another
 *   rank, so several ranks may share one GPU.  Callbacks return 0 on success
 *   (else the call fails with PEEL_ENCCL) and must be collective: every rank
 *   calls them in the same order.
 *     allreduce(ctx, vals, count): vals[count] (host u64) <- elementwise sum.
 *     allgather(ctx, send, recv, bytes): recv[P bytes] <- each rank's send[bytes].
 *     alltoallv(ctx, send, sbytes[P], recv, rbytes[P]): rank me sends sbytes[d]
 *       bytes to every rank d (segments packed in increasing d in send; sbytes[me]
 *       = 0) and receives rbytes[q] bytes from every q, packed in increasing q.
 * Errors (all partitioned calls): a rank that fails locally keeps taking part in
 *   the collectives with an error word set; every rank then leaves at the same
 *   collective -- the failing rank with its status, the others with PEEL_EPEER --
 *   so no rank is left blocked in a collective.  A rank that dies or disappears
 *   cannot do that: NCCL communicators wait on their streams with a watchdog
 *   (asynchronous NCCL errors, or PEEL_NCCL_TIMEOUT_S seconds, default 600), which
 *   aborts the communicator and returns PEEL_ENCCL; every later call on an aborted
 *   communicator returns PEEL_ENCCL (destroy it and create a new one).
 * peel_kcore_dist: edges dev u32 [m][r] (replicated); core_mask dev u8: the
 *   rank's slice [v1 - v0] (NCCL) or all n (virtual); rounds/survivors/killed
 *   host, global (identical on every rank); workspace dev,
 *   peel_kcore_dist_workspace_bytes bytes (per rank; virtual: all shards).
 *   Blocking (host-driven rounds: two stream syncs per round).
 */
typedef struct peel_comm peel_comm;
typedef int (*peel_host_allreduce_fn)(void *ctx, uint64_t *vals, uint64_t count);
typedef int (*peel_host_allgather_fn)(void *ctx, const void *send, void *recv, uint64_t bytes);
typedef int (*peel_host_alltoallv_fn)(void *ctx, const void *send, const uint64_t *sbytes, void *recv,
                                      const uint64_t *rbytes);
peel_status peel_comm_unique_id(void *id128);
peel_status peel_comm_init(const void *id128, int nranks, int rank, peel_comm **out);
peel_status peel_comm_init_host(int nranks, int rank, peel_host_allreduce_fn allreduce,
                                peel_host_allgather_fn allgather, peel_host_alltoallv_fn alltoallv, void *ctx,
                                peel_comm **out);
peel_status peel_comm_init_virtual(int nshards, peel_comm **out);
void peel_comm_destroy(peel_comm *c);
size_t peel_kcore_dist_workspace_bytes(const peel_comm *c, uint64_t n, uint64_t m, uint32_t r, uint32_t k);
peel_status peel_kcore_dist(peel_comm *c, const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r, uint32_t k,
                            uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors, uint64_t *killed,
                            uint32_t cap, void *workspace, size_t ws_bytes, void *stream);

/* ======================================================================= */
/* IBLT -- cells {count, checksum, key} with XOR accumulators   */
/* ======================================================================= */

/*
 * Cell layout in device memory (16 bytes, 16-byte aligned, array of structs):
 *   struct { uint32_t count; uint32_t hashSum; uint64_t keySum; }
 * keySum / hashSum are the paper's key and checksum fields,
 * XOR accumulators; count is this build's count field (signed, two's
 * complement), which makes "pure" exact: count == 1 and
 * hashSum == checkSum(keySum).  The table and all peel scratch live
 * in caller-owned device memory `mem` of iblt_mem_bytes(cells, r) bytes; the
 * cell array is at offset 0.
 *
 * Hashes: seed_h = mix64((seed ^ 0x6A09E667F3BCC909) + G),
 * seed_c = mix64((seed ^ 0xBB67AE8584CAA73B) + G), G = 0x9E3779B97F4A7C15;
 * cell j-th candidate = umulhi64(mix64(x ^ seed_h ^ (j+1)*0xD1B54A32D192ED03), cells),
 * duplicates rejected, until r distinct cells; checkSum(x) = mix64(x ^ seed_c) >> 32.
 */
typedef struct peel_iblt peel_iblt;

size_t iblt_mem_bytes(uint64_t cells, uint32_t r);

/* Zero the cells and create the handle.  EINVAL: r < 2, r > 8, cells < r,
 * cells >= 2^32, mem NULL, mem_bytes too small, mem not 16-byte aligned. */
peel_status iblt_build(uint64_t cells, uint32_t r, uint64_t seed, void *mem, size_t mem_bytes,
                       void *stream, peel_iblt **out);

/* IBLT_FLAG_SUBTABLES -- the paper's GPU layout: the table is split into r
 * subtables of cells / r cells (r must divide cells) and key x goes to ONE cell per
 * subtable, h_j(x) = j cells/r + umulhi64(mix64(x ^ seed_h ^ (j+1) 0xD1B54A32D192ED03), cells/r).
 * iblt_peel on such a table runs the paper's schedule: each round iterates the r subtables
 * serially, recovering all pure cells of subtable j in parallel; `rounds` is then the
 * flattened index of the last subtable step that recovered a key and per_round[s-1] the
 * keys recovered at step s. */
#define IBLT_FLAG_SUBTABLES 1u
/* IBLT_FLAG_BLOCKED -- locality-aware hashing, the paper's open question (
 * DESIGN.md reading R27): the table is nb blocks of B = 2^blog cells (B must divide cells,
 * r <= B; blog = IBLT_BLOCK_LOG(flags), 0 meaning 16) and all r cells of key x lie in one
 * block: b = umulhi64(mix64(x ^ seed_h ^ 0x9E6C63D0676A9A99), cells / B), cell j =
 * b B + the j-th cell of the plain hash over B cells.  Recovery is the plain
 * round-synchronous schedule; a block's cells are contiguous, so a round's atomics for the
 * frontier entries in flight stay in a few blocks. */
#define IBLT_FLAG_BLOCKED 2u
#define IBLT_BLOCK_LOG_SHIFT 8
#define IBLT_BLOCK_LOG(flags) (((flags) >> IBLT_BLOCK_LOG_SHIFT) & 0xFFu)
peel_status iblt_build_ex(uint64_t cells, uint32_t r, uint64_t seed, uint32_t flags, void *mem,
                          size_t mem_bytes, void *stream, peel_iblt **out);

/* Insert nkeys keys (dev u64): XOR x into keySum and checkSum(x) into
 * hashSum of each of x's r cells, count += 1 (one thread per key
 * with atomic XOR).  Keys must be distinct and not already in the
 * table (XOR would cancel them; caller error, not detected). */
peel_status iblt_insert(peel_iblt *t, const uint64_t *keys, uint64_t nkeys, void *stream);

/* Delete: the same XOR update with count -= 1 ("insertion and deletion
 * procedures are identical"). */
peel_status iblt_delete(peel_iblt *t, const uint64_t *keys, uint64_t nkeys, void *stream);

/*
 * iblt_peel -- round-synchronous recovery (the 2-core peel of the
 * IBLT's hypergraph).  Each round snapshots the pure cells, recovers
 * each of their keys exactly once (the owner is the round-start-pure cell
 * with the lowest hash index among the key's cells), deletes every recovered
 * key from its r cells, and stops at the first round recovering nothing.
 * DESTRUCTIVE: the table holds the unrecovered remainder afterwards.
 * A table that has only seen iblt_insert since iblt_build (no iblt_delete, no
 * iblt_subtract into it, no iblt_cells) is insert-only: its counts are the true
 * key counts, so the owner's pure cell is zeroed with one store instead of an
 * XOR-delete.  The result is identical either way.
 * out: out_keys dev u64 [cap_keys], recovered keys in unspecified order;
 *      nrecovered host u64 (may exceed cap_keys: then PEEL_ETRUNC and only
 *      cap_keys were stored); rounds host u32; per_round host u64 [cap]
 *      (nullable) keys recovered in round t; complete host int (nullable):
 *      1 iff every cell is zero afterwards (success iff the 2-core is empty) --
 *      for an insert-only table (no delete, subtract or raw cell access since
 *      the build) decided as "every inserted key was recovered", which is the
 *      same condition, without scanning the cells.
 * Blocking.
 */
peel_status iblt_peel(peel_iblt *t, uint64_t *out_keys, uint64_t cap_keys, uint64_t *nrecovered,
                      uint32_t *rounds, uint64_t *per_round, uint32_t cap, int *complete,
                      void *stream);

/* Set difference (the sparse-recovery use of P:476-480): a <- a - b cell-wise
 * (count subtracts, key and checksum fields XOR) -- the IBLT of the signed multiset A - B.
 * Both tables must have equal cells, r, seed and layout (else EINVAL).  Stream-ordered. */
peel_status iblt_subtract(peel_iblt *a, const peel_iblt *b, void *stream);

/* iblt_peel for signed tables: a cell is pure when count is +1 or -1 and hashSum ==
 * checkSum(keySum); a recovered key is removed with the opposite sign.  out_sign dev
 * int8 [cap_keys]: +1 for keys only in A, -1 for keys only in B.  Other arguments and
 * the result as iblt_peel.  EINVAL on a subtable table. */
peel_status iblt_peel_signed(peel_iblt *t, uint64_t *out_keys, int8_t *out_sign, uint64_t cap_keys,
                             uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round, uint32_t cap,
                             int *complete, void *stream);

/* Device pointer to the 16-byte cell array (for tests and serialisation).  The pointer
 * is writable, so the call marks the table as no longer insert-only: later iblt_peel
 * calls take the general path (three atomics per cell of a recovered key) instead of
 * clearing round-start-pure cells with a plain store.  iblt_delete and iblt_subtract
 * (on a) do the same. */
void *iblt_cells(const peel_iblt *t);

/* edges[i][j] (dev u32 [nkeys][r]) = j-th cell of keys[i]: the IBLT's
 * hypergraph, cells = vertices, keys = edges. */
peel_status iblt_to_hypergraph(const peel_iblt *t, const uint64_t *keys, uint64_t nkeys,
                               uint32_t *edges, void *stream);

/* Free the handle (not the caller's memory). */
void iblt_destroy(peel_iblt *t);

/* ---- cell-partitioned IBLT over P GPUs ------------------------------------
 * One table of `cells` cells split by cell range over the communicator's P shards (ranks, or
 * virtual shards of one GPU): shard q owns cells [q cs, (q+1) cs), cs = ceil(cells/P)
 * rounded up to 32.  iblt_dist_recover inserts the nkeys keys (dev u64, the SAME array on
 * every rank: each shard applies them to its own cells) and runs the round-synchronous
 * recovery of iblt_peel: per round the shards gather each other's round-start pure cells
 * (one allgather of a cells-bit bitmap), each key is found by the shard owning its
 * lowest-index pure cell (the owner rule) and sent to the shards owning its cells, which
 * XOR-delete it; then candidates are re-tested.  Results equal iblt_peel on one table.
 * flags: 0 or IBLT_FLAG_BLOCKED (+ IBLT_BLOCK_LOG); seed, hashes as iblt_build.
 * Outputs: out_keys (dev u64, cap_keys) receives the keys found by THIS rank (virtual: all
 * shards), *nrecovered their number; rounds, per_round[0 .. min(rounds, cap)) (host, keys
 * recovered per round over all shards) and *complete (all cells of all shards zero) are
 * global.  mem: dev, iblt_dist_mem_bytes(c, cells, r) bytes (per rank; virtual: all shards).
 * Collective over the communicator's ranks; blocking.  EINVAL: bad shape or flags (r in
 * [2, 8], P <= 8); ENOMEM: mem too small; ETRUNC: cap_keys or cap exceeded, or 65536
 * rounds; ENCCL; EPEER.
 * iblt_dist_recover_cells: the same recovery of an EXISTING table: cells_in (dev, `cells`
 * 16-byte cells laid out as iblt_cells() returns them -- e.g. a subtracted, deserialized or
 * received table; the same bytes on every rank) instead of keys to insert; each shard copies
 * its own cell range.  Unsigned recovery (count +1).  R28: a cell is pure when
 * its count is 1, its checksum matches and it is one of its key's cells. */
size_t iblt_dist_mem_bytes(const peel_comm *c, uint64_t cells, uint32_t r);
peel_status iblt_dist_recover_cells(peel_comm *c, const void *cells_in, uint64_t cells, uint32_t r, uint64_t seed,
                                    uint32_t flags, uint64_t *out_keys, uint64_t cap_keys, uint64_t *nrecovered,
                                    uint32_t *rounds, uint64_t *per_round, uint32_t cap, int *complete, void *mem,
                                    size_t mem_bytes, void *stream);
peel_status iblt_dist_recover(peel_comm *c, uint64_t cells, uint32_t r, uint64_t seed, uint32_t flags,
                              const uint64_t *keys, uint64_t nkeys, uint64_t *out_keys, uint64_t cap_keys,
                              uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round, uint32_t cap,
                              int *complete, void *mem, size_t mem_bytes, void *stream);

/* ======================================================================= */
/* Measurement support                                                      */
/* ======================================================================= */

/*
 * When enabled, every library call records a CUDA event pair on `stream`
 * around each kernel it launches.  Blocking calls (peel_kcore, iblt_peel)
 * resolve them: afterwards peel_profile_read returns up to `cap` (name,
 * milliseconds, launches) triples for every launch since the previous blocking
 * call (e.g. iblt_insert + iblt_peel), in first-launch order.  Names are static
 * strings.  Returns the number of entries.  Disabled by default.
 */
void peel_profile_enable(int on);
int peel_profile_read(const char **names, double *ms, uint32_t *launches, int cap);
/* Kernel launches since the previous blocking call, counted through the last
 * blocking call (always counted, profiling or not). */
uint32_t peel_last_launches(void);
/* With profiling enabled: per-round device time (ms, from %globaltimer at each
 * round barrier) of the last peel_kcore call; returns the number of rounds. */
int peel_profile_rounds(double *ms, uint32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* PEEL_H_ */
