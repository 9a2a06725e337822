/*
 * peel_oracle.c -- CPU ORACLE for parallel peeling (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the plain, slow, single-threaded reference that the CUDA path is
 * checked against.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product library
 * (paper_1302_7014_b200/) never includes, links or calls anything in oracle/,
 * and this file includes nothing from the product tree.
 *
 * Citations: "P:n" = line n of the paper (arXiv 1302.7014, PAPER.md);
 * "S:n" = line n of SPEC.md; "SURVEY §8 c3" = the hash/generator definitions
 * this build adopts (docs restated in DESIGN.md §3).
 *
 * Every function follows the plain definition, in the paper's order:
 *   - ora_philox4x32_10 ........ Random123 Philox4x32-10 block function (KAT-pinned)
 *   - ora_gen_edge ............. G^r_{n,cn}: edge e = r distinct vertices
 *   - ora_sync_peel ............ round-synchronous peel, literal
 *   - ora_queue_peel ........... serial greedy peel
 *   - ora_gen_partitioned ...... the subtable hypergraph model
 *   - ora_subround_peel ........ the subround (subtable) peel
 *   - ora_iblt_* ............... IBLT insert / round-synchronous recovery
 *   - ora_iblt_serial_recover .. one-pure-cell-at-a-time recovery
 *   - ora_cells_of_blocked ..... blocked (locality-aware) hashing, the paper's open question
 * Nothing here is blocked, fused or reordered beyond what the definitions state.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Counter-based PRF: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11;       */
/* Random123).  Pinned by the Random123 known-answer vectors in tests.        */
/* ------------------------------------------------------------------------- */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void ora_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int i = 0; i < 10; i++) {
        if (i > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* high 64 bits of the 128-bit product (fastrange64 of a 64-bit draw onto [0,n)) */
static uint64_t umulhi64(uint64_t a, uint64_t b) {
    return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
}

/* ------------------------------------------------------------------------- */
/* a1: the hypergraph G^r_{n,cn} ("cn hyperedges, where each         */
/* hyperedge consists of r distinct vertices"; "each edge is chosen    */
/* independently and uniformly").  Draw j of edge e is half (j%2) of Philox   */
/* block (ctr = e_lo, e_hi, j/2, 'EDGE'; key = seed_lo, seed_hi); a draw d is */
/* mapped to vertex umulhi64(d, n) and rejected if already in the edge.       */
/* ------------------------------------------------------------------------- */
#define ORA_EDGE_TAG 0x45444745u /* 'EDGE' */

int ora_gen_edge(uint64_t seed, uint64_t n, uint32_t r, uint64_t e, uint32_t *out) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t accepted = 0;
    uint32_t w[4];
    for (uint32_t j = 0; accepted < r; j++) {
        if (j % 2 == 0) {
            uint32_t ctr[4] = {(uint32_t)e, (uint32_t)(e >> 32), j / 2, ORA_EDGE_TAG};
            ora_philox4x32_10(ctr, key, w);
        }
        uint64_t d = (j % 2 == 0) ? (((uint64_t)w[1] << 32) | w[0])
                                  : (((uint64_t)w[3] << 32) | w[2]);
        uint32_t v = (uint32_t)umulhi64(d, n);
        int dup = 0;
        for (uint32_t i = 0; i < accepted; i++)
            if (out[i] == v) dup = 1;
        if (!dup) out[accepted++] = v;
        if (j > 100000) return -1; /* n < r cannot terminate; caller validates */
    }
    return 0;
}

int ora_gen_hypergraph(uint64_t seed, uint64_t n, uint64_t m, uint32_t r, uint32_t *edges) {
    if (r < 2 || n < r) return -1;
    for (uint64_t e = 0; e < m; e++)
        if (ora_gen_edge(seed, n, r, e, edges + e * r)) return -1;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* The subtable (r-partite) model: vertices are split into r      */
/* classes of size n/r, class j = [j n/r, (j+1) n/r), and every edge has     */
/* exactly one vertex in each class, chosen independently and uniformly.     */
/* The vertex of class j is draw j (half j%2 of Philox block j/2, tag 'SUBT') */
/* mapped by umulhi64 onto the class; no rejection is needed.                */
/* ------------------------------------------------------------------------- */
#define ORA_SUBT_TAG 0x53554254u /* 'SUBT' */

int ora_gen_partitioned(uint64_t seed, uint64_t n, uint64_t m, uint32_t r, uint32_t *edges) {
    if (r < 2 || n < r || n % r) return -1;
    uint64_t s = n / r;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    for (uint64_t e = 0; e < m; e++)
        for (uint32_t j = 0; j < r; j++) {
            if (j % 2 == 0) {
                uint32_t ctr[4] = {(uint32_t)e, (uint32_t)(e >> 32), j / 2, ORA_SUBT_TAG};
                ora_philox4x32_10(ctr, key, w);
            }
            uint64_t d = (j % 2 == 0) ? (((uint64_t)w[1] << 32) | w[0]) : (((uint64_t)w[3] << 32) | w[2]);
            edges[e * r + j] = (uint32_t)(j * s + umulhi64(d, s));
        }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* SplitMix64 (Steele, Lea, Flood, OOPSLA'14) finalizer, used for the IBLT    */
/* keys, the r cell hashes h_1..h_r and checkSum ("r hash          */
/* functions", "checkSum is some simple pseudorandom function").             */
/* ------------------------------------------------------------------------- */
#define ORA_GAMMA 0x9E3779B97F4A7C15ull

uint64_t ora_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* key_i = i-th output of a SplitMix64 stream started at state `seed` */
void ora_gen_keys(uint64_t seed, uint64_t nkeys, uint64_t *keys) {
    for (uint64_t i = 0; i < nkeys; i++) keys[i] = ora_mix64(seed + (i + 1) * ORA_GAMMA);
}

uint64_t ora_seed_h(uint64_t seed) { return ora_mix64((seed ^ 0x6A09E667F3BCC909ull) + ORA_GAMMA); }
uint64_t ora_seed_c(uint64_t seed) { return ora_mix64((seed ^ 0xBB67AE8584CAA73Bull) + ORA_GAMMA); }

/* checkSum(x) */
uint32_t ora_checksum(uint64_t x, uint64_t seed_c) { return (uint32_t)(ora_mix64(x ^ seed_c) >> 32); }

/* the r distinct cells h_1(x)..h_r(x) in [0, C) */
int ora_cells_of(uint64_t x, uint64_t C, uint32_t r, uint64_t seed_h, uint64_t *out) {
    uint32_t accepted = 0;
    for (uint64_t j = 0; accepted < r; j++) {
        uint64_t z = ora_mix64(x ^ seed_h ^ ((j + 1) * 0xD1B54A32D192ED03ull));
        uint64_t c = umulhi64(z, C);
        int dup = 0;
        for (uint32_t i = 0; i < accepted; i++)
            if (out[i] == c) dup = 1;
        if (!dup) out[accepted++] = c;
        if (j > 100000) return -1;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Round-synchronous parallel peel, written literally ("in each      */
/* round, all vertices of degree less than k and their adjacent edges are     */
/* removed in parallel"; an edge is peeled if some adjacent vertex */
/* is peeled).  Round t snapshots F_t = {alive v : deg(v) < k} (deg 0         */
/* included), removes F_t, then scans every alive edge and kills those with   */
/* an endpoint in F_t.  rounds = number of rounds with F_t non-empty (the     */
/* terminal empty scan is not counted).  O((n+m) * rounds) by design.         */
/*                                                                            */
/* outputs: core_mask[n] (1 = in the k-core), *rounds, survivors[t-1] =       */
/* alive vertices after round t, killed[t-1] = edges killed in round t,       */
/* peel_round[v] = round v was removed in (0 = never; optional).              */
/* returns 0, or 1 if more than cap rounds (first cap entries written),      */
/* or -1 on allocation failure / bad input.                                   */
/* ------------------------------------------------------------------------- */
int ora_sync_peel(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r, uint32_t k,
                  uint8_t *core_mask, uint32_t *rounds, uint64_t *survivors, uint64_t *killed,
                  uint32_t cap, uint32_t *peel_round) {
    int64_t *deg = (int64_t *)calloc(n ? n : 1, sizeof(int64_t));
    uint8_t *alive_v = (uint8_t *)malloc(n ? n : 1);
    uint8_t *alive_e = (uint8_t *)malloc(m ? m : 1);
    uint8_t *inF = (uint8_t *)calloc(n ? n : 1, 1);
    uint64_t *F = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!deg || !alive_v || !alive_e || !inF || !F) {
        free(deg); free(alive_v); free(alive_e); free(inF); free(F);
        return -1;
    }
    for (uint64_t e = 0; e < m; e++)
        for (uint32_t j = 0; j < r; j++) {
            uint32_t u = edges[e * r + j];
            if (u >= n) { free(deg); free(alive_v); free(alive_e); free(inF); free(F); return -1; }
            deg[u] += 1;
        }
    memset(alive_v, 1, n);
    memset(alive_e, 1, m);
    if (peel_round) memset(peel_round, 0, n * sizeof(uint32_t));
    uint32_t t = 0;
    uint64_t surv = n;
    int status = 0;
    for (;;) {
        uint64_t nF = 0;
        for (uint64_t v = 0; v < n; v++)
            if (alive_v[v] && deg[v] < (int64_t)k) F[nF++] = v;
        if (nF == 0) break;
        t += 1;
        for (uint64_t i = 0; i < nF; i++) {
            alive_v[F[i]] = 0;
            inF[F[i]] = 1;
            if (peel_round) peel_round[F[i]] = t;
        }
        uint64_t nkill = 0;
        for (uint64_t e = 0; e < m; e++) {
            if (!alive_e[e]) continue;
            int hit = 0;
            for (uint32_t j = 0; j < r; j++)
                if (inF[edges[e * r + j]]) hit = 1;
            if (hit) {
                alive_e[e] = 0;
                nkill++;
                for (uint32_t j = 0; j < r; j++) deg[edges[e * r + j]] -= 1;
            }
        }
        for (uint64_t i = 0; i < nF; i++) inF[F[i]] = 0;
        surv -= nF;
        if (t <= cap) {
            if (survivors) survivors[t - 1] = surv;
            if (killed) killed[t - 1] = nkill;
        } else {
            status = 1;
        }
    }
    *rounds = t;
    for (uint64_t v = 0; v < n; v++) core_mask[v] = alive_v[v];
    free(deg); free(alive_v); free(alive_e); free(inF); free(F);
    return status;
}

/* ------------------------------------------------------------------------- */
/* Subround peel: vertices in r classes [j n/r, (j+1) n/r);       */
/* round i = r subrounds, and subround j removes every alive vertex of class */
/* j whose degree is < k at the START of the subround (a snapshot), together */
/* with its alive edges, after subrounds 1..j-1 of the same round applied.   */
/* Stops after the first full round that removes nothing.  Written           */
/* literally: each subround scans the class and then every alive edge.      */
/* outputs: core_mask, *subrounds = flattened index (i-1) r + j of the last  */
/* subround that removed a vertex, *rounds = rounds with a removal,          */
/* survivors[s-1] = alive vertices after flattened subround s (s =           */
/* 1..subrounds), killed[s-1] = edges killed there (nullable).  returns 0, 1 */
/* if subrounds > cap, -1 on bad input/alloc.                                */
/* ------------------------------------------------------------------------- */
int ora_subround_peel(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r, uint32_t k,
                      uint8_t *core_mask, uint32_t *rounds, uint32_t *subrounds,
                      uint64_t *survivors, uint64_t *killed, uint32_t cap) {
    if (r < 2 || n % r) return -1;
    uint64_t cs = n / r;
    int64_t *deg = (int64_t *)calloc(n ? n : 1, sizeof(int64_t));
    uint8_t *alive_v = (uint8_t *)malloc(n ? n : 1);
    uint8_t *alive_e = (uint8_t *)malloc(m ? m : 1);
    uint8_t *inF = (uint8_t *)calloc(n ? n : 1, 1);
    uint64_t *F = (uint64_t *)malloc((cs ? cs : 1) * sizeof(uint64_t));
    if (!deg || !alive_v || !alive_e || !inF || !F) {
        free(deg); free(alive_v); free(alive_e); free(inF); free(F);
        return -1;
    }
    for (uint64_t e = 0; e < m * r; e++) {
        if (edges[e] >= n) { free(deg); free(alive_v); free(alive_e); free(inF); free(F); return -1; }
        deg[edges[e]] += 1;
    }
    memset(alive_v, 1, n);
    memset(alive_e, 1, m);
    uint64_t surv = n, flat = 0, last = 0;
    uint32_t nrounds = 0;
    int status = 0;
    for (uint32_t i = 1;; i++) {
        int any = 0;
        for (uint32_t j = 0; j < r; j++) {
            flat++;
            uint64_t nF = 0, nkill = 0;
            for (uint64_t v = j * cs; v < (j + 1) * cs; v++)
                if (alive_v[v] && deg[v] < (int64_t)k) F[nF++] = v;
            if (nF) {
                for (uint64_t q = 0; q < nF; q++) { alive_v[F[q]] = 0; inF[F[q]] = 1; }
                for (uint64_t e = 0; e < m; e++) {
                    if (!alive_e[e]) continue;
                    int hit = 0;
                    for (uint32_t t = 0; t < r; t++)
                        if (inF[edges[e * r + t]]) hit = 1;
                    if (hit) {
                        alive_e[e] = 0;
                        nkill++;
                        for (uint32_t t = 0; t < r; t++) deg[edges[e * r + t]] -= 1;
                    }
                }
                for (uint64_t q = 0; q < nF; q++) inF[F[q]] = 0;
                surv -= nF;
                any = 1;
                last = flat;
            }
            if (flat <= cap) {
                survivors[flat - 1] = surv;
                if (killed) killed[flat - 1] = nkill;
            } else if (nF) status = 1;
        }
        if (!any) break;
        nrounds = i;
    }
    *rounds = nrounds;
    *subrounds = (uint32_t)last;
    for (uint64_t v = 0; v < n; v++) core_mask[v] = alive_v[v];
    free(deg); free(alive_v); free(alive_e); free(inF); free(F);
    return status;
}

/* ------------------------------------------------------------------------- */
/* Serial greedy peel ("vertices with degree less than k are */
/* repeatedly removed, together with their associated edges").  Queue-driven, */
/* one vertex at a time; a different algorithm that must reach the same      */
/* unique k-core.  Output: core_mask only.                 */
/* ------------------------------------------------------------------------- */
int ora_queue_peel(const uint32_t *edges, uint64_t n, uint64_t m, uint32_t r, uint32_t k,
                   uint8_t *core_mask) {
    uint64_t *off = (uint64_t *)calloc(n + 1, sizeof(uint64_t));
    int64_t *deg = (int64_t *)calloc(n ? n : 1, sizeof(int64_t));
    uint64_t *adj = (uint64_t *)malloc((m * r ? m * r : 1) * sizeof(uint64_t));
    uint8_t *alive_e = (uint8_t *)malloc(m ? m : 1);
    uint8_t *queued = (uint8_t *)calloc(n ? n : 1, 1);
    uint64_t *queue = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!off || !deg || !adj || !alive_e || !queued || !queue) {
        free(off); free(deg); free(adj); free(alive_e); free(queued); free(queue);
        return -1;
    }
    for (uint64_t e = 0; e < m * r; e++) off[edges[e] + 1] += 1;
    for (uint64_t v = 0; v < n; v++) off[v + 1] += off[v];
    uint64_t *fill = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!fill) { free(off); free(deg); free(adj); free(alive_e); free(queued); free(queue); return -1; }
    for (uint64_t v = 0; v < n; v++) fill[v] = off[v];
    for (uint64_t e = 0; e < m; e++)
        for (uint32_t j = 0; j < r; j++) {
            uint32_t u = edges[e * r + j];
            adj[fill[u]++] = e;
            deg[u] += 1;
        }
    free(fill);
    memset(alive_e, 1, m);
    uint64_t head = 0, tail = 0;
    for (uint64_t v = 0; v < n; v++)
        if (deg[v] < (int64_t)k) { queue[tail++] = v; queued[v] = 1; }
    while (head < tail) {
        uint64_t v = queue[head++];
        for (uint64_t p = off[v]; p < off[v + 1]; p++) {
            uint64_t e = adj[p];
            if (!alive_e[e]) continue;
            alive_e[e] = 0;
            for (uint32_t j = 0; j < r; j++) {
                uint32_t u = edges[e * r + j];
                deg[u] -= 1;
                if (!queued[u] && deg[u] < (int64_t)k) { queue[tail++] = u; queued[u] = 1; }
            }
        }
    }
    for (uint64_t v = 0; v < n; v++) core_mask[v] = queued[v] ? 0 : 1;
    free(off); free(deg); free(adj); free(alive_e); free(queued); free(queue);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* IBLT.  Cell = {count, keySum, hashSum}; insert XORs x into the */
/* key field and checkSum(x) into the checksum field of each of x's r cells   */
/* and counts it (this build's count field, reading R8).*/
/* ------------------------------------------------------------------------- */
typedef struct {
    uint64_t C;
    uint32_t r;
    int subtables; /* 1: r subtables of C/r cells, one cell per subtable per key */
    uint32_t blog; /* > 0: blocked hashing, all r cells in one block of 2^blog cells (R27) */
    uint64_t seed_h, seed_c;
    int64_t *count;
    uint64_t *keySum;
    uint32_t *hashSum;
} ora_iblt;

ora_iblt *ora_iblt_new_ex(uint64_t C, uint32_t r, uint64_t seed, int subtables) {
    if (r < 2 || C < r || (subtables && C % r)) return NULL;
    ora_iblt *t = (ora_iblt *)calloc(1, sizeof(ora_iblt));
    if (!t) return NULL;
    t->C = C; t->r = r; t->subtables = subtables;
    t->seed_h = ora_seed_h(seed);
    t->seed_c = ora_seed_c(seed);
    t->count = (int64_t *)calloc(C, sizeof(int64_t));
    t->keySum = (uint64_t *)calloc(C, sizeof(uint64_t));
    t->hashSum = (uint32_t *)calloc(C, sizeof(uint32_t));
    if (!t->count || !t->keySum || !t->hashSum) {
        free(t->count); free(t->keySum); free(t->hashSum); free(t);
        return NULL;
    }
    return t;
}

ora_iblt *ora_iblt_new(uint64_t C, uint32_t r, uint64_t seed) { return ora_iblt_new_ex(C, r, seed, 0); }

/* blocked table: C = nb 2^blog cells (R27) */
ora_iblt *ora_iblt_new_blocked(uint64_t C, uint32_t r, uint64_t seed, uint32_t blog) {
    if (blog < 4 || blog > 30 || C % (1ull << blog) || r > (1u << blog)) return NULL;
    ora_iblt *t = ora_iblt_new_ex(C, r, seed, 0);
    if (t) t->blog = blog;
    return t;
}

/* Blocked hashing (locality-aware hashing, the paper's open question P:706-708; DESIGN.md
 * reading R27): the key's block b = umulhi64(mix64(x ^ seed_h ^ 0x9E6C63D0676A9A99), C / B)
 * with B = 2^blog, then r distinct cells of [b B, (b+1) B) drawn exactly as ora_cells_of
 * draws them from [0, C) -- the same draws j = 0, 1, ... mapped into B cells instead of C. */
int ora_cells_of_blocked(uint64_t x, uint64_t C, uint32_t r, uint64_t seed_h, uint32_t blog, uint64_t *out) {
    const uint64_t B = 1ull << blog;
    const uint64_t b = umulhi64(ora_mix64(x ^ seed_h ^ 0x9E6C63D0676A9A99ull), C / B);
    if (ora_cells_of(x, B, r, seed_h, out) != 0) return -1;
    for (uint32_t j = 0; j < r; j++) out[j] += b * B;
    return 0;
}

/* subtable hashing ("hash each item into one cell in each subtable"):  */
/* h_j(x) = j C/r + umulhi64(mix64(x ^ seed_h ^ (j+1) 0xD1B54A32D192ED03), C/r) */
void ora_cells_of_subtable(uint64_t x, uint64_t C, uint32_t r, uint64_t seed_h, uint64_t *out) {
    uint64_t s = C / r;
    for (uint32_t j = 0; j < r; j++)
        out[j] = j * s + umulhi64(ora_mix64(x ^ seed_h ^ ((j + 1) * 0xD1B54A32D192ED03ull)), s);
}

static void key_cells(const ora_iblt *t, uint64_t x, uint64_t *cells) {
    if (t->subtables) ora_cells_of_subtable(x, t->C, t->r, t->seed_h, cells);
    else if (t->blog) ora_cells_of_blocked(x, t->C, t->r, t->seed_h, t->blog, cells);
    else ora_cells_of(x, t->C, t->r, t->seed_h, cells);
}

void ora_iblt_free(ora_iblt *t) {
    if (!t) return;
    free(t->count); free(t->keySum); free(t->hashSum); free(t);
}

uint64_t ora_iblt_seed_h(const ora_iblt *t) { return t->seed_h; }
uint64_t ora_iblt_seed_c(const ora_iblt *t) { return t->seed_c; }

/* sign = +1 insert, -1 delete ("the insertion and deletion procedures are identical") */
static void iblt_apply(ora_iblt *t, uint64_t x, int sign) {
    uint64_t cells[16];
    key_cells(t, x, cells);
    uint32_t h = ora_checksum(x, t->seed_c);
    for (uint32_t j = 0; j < t->r; j++) {
        t->count[cells[j]] += sign;
        t->keySum[cells[j]] ^= x;
        t->hashSum[cells[j]] ^= h;
    }
}

int ora_iblt_insert(ora_iblt *t, const uint64_t *keys, uint64_t nkeys) {
    if (t->r > 16) return -1;
    for (uint64_t i = 0; i < nkeys; i++) iblt_apply(t, keys[i], +1);
    return 0;
}

int ora_iblt_delete(ora_iblt *t, const uint64_t *keys, uint64_t nkeys) {
    if (t->r > 16) return -1;
    for (uint64_t i = 0; i < nkeys; i++) iblt_apply(t, keys[i], -1);
    return 0;
}

void ora_iblt_dump(const ora_iblt *t, int64_t *count, uint64_t *keySum, uint32_t *hashSum) {
    memcpy(count, t->count, t->C * sizeof(int64_t));
    memcpy(keySum, t->keySum, t->C * sizeof(uint64_t));
    memcpy(hashSum, t->hashSum, t->C * sizeof(uint32_t));
}

/* Overwrite every cell (a serialized table; tests also forge cells with it). */
void ora_iblt_load(ora_iblt *t, const int64_t *count, const uint64_t *keySum, const uint32_t *hashSum) {
    memcpy(t->count, count, t->C * sizeof(int64_t));
    memcpy(t->keySum, keySum, t->C * sizeof(uint64_t));
    memcpy(t->hashSum, hashSum, t->C * sizeof(uint32_t));
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* A pure cell "only contain[s] one item", x = its key field.  This   */
/* build's test (reading R28): count == 1, the checksum field       */
/* equals checkSum(x), and c is one of x's own cells h_1(x) ..    */
/* h_r(x) -- a cell holding only x is necessarily one of x's     */
/* cells, so a cell failing that test holds more than one item whatever its   */
/* other fields say (a checksum collision, a forged or corrupted table).      */
static int cell_of_key(const ora_iblt *t, uint64_t c, uint64_t x) {
    uint64_t cells[16];
    key_cells(t, x, cells);
    for (uint32_t j = 0; j < t->r; j++)
        if (cells[j] == c) return 1;
    return 0;
}

static int iblt_pure(const ora_iblt *t, uint64_t c) {
    return t->count[c] == 1 && t->hashSum[c] == ora_checksum(t->keySum[c], t->seed_c) &&
           cell_of_key(t, c, t->keySum[c]);
}

/* At most this many rounds (steps, for the subtable schedule) are run; a     */
/* table still holding pure cells after the last one is reported truncated    */
/* (status 1).  Forged signed tables are not known to terminate (DESIGN R28). */
#define ORA_IBLT_ROUND_LIMIT 65536u

/* Round-synchronous recovery: each round snapshots the set of    */
/* pure cells, recovers the SET of their keys (set semantics: a key seen in   */
/* several pure cells is recovered once), deletes every recovered  */
/* key from its r cells, and stops at the first round recovering nothing.    */
/* Destructive.  out_keys[] in recovery order (per round ascending).          */
/* returns 0; 1 if rounds > cap or keys > cap_keys (truncated); -1 on alloc.  */
int ora_iblt_peel(ora_iblt *t, uint64_t *out_keys, uint64_t cap_keys, uint64_t *nrecovered,
                  uint32_t *rounds, uint64_t *per_round, uint32_t cap, int *complete) {
    uint64_t C = t->C;
    uint64_t *X = (uint64_t *)malloc(C * sizeof(uint64_t));
    if (!X) return -1;
    uint64_t nrec = 0;
    uint32_t rt = 0;
    int status = 0;
    for (;;) {
        uint64_t nX = 0;
        for (uint64_t c = 0; c < C; c++)
            if (iblt_pure(t, c)) X[nX++] = t->keySum[c];
        if (nX == 0) break;
        if (rt == ORA_IBLT_ROUND_LIMIT) { status = 1; break; }
        qsort(X, nX, sizeof(uint64_t), cmp_u64);
        uint64_t u = 0;
        for (uint64_t i = 0; i < nX; i++)
            if (i == 0 || X[i] != X[i - 1]) X[u++] = X[i];
        nX = u;
        rt += 1;
        for (uint64_t i = 0; i < nX; i++) {
            iblt_apply(t, X[i], -1);
            if (nrec < cap_keys) out_keys[nrec] = X[i]; else status = 1;
            nrec++;
        }
        if (rt <= cap) per_round[rt - 1] = nX; else status = 1;
    }
    free(X);
    *nrecovered = nrec;
    *rounds = rt;
    int z = 1;
    for (uint64_t c = 0; c < C; c++)
        if (t->count[c] != 0 || t->keySum[c] != 0 || t->hashSum[c] != 0) { z = 0; break; }
    *complete = z;
    return status;
}

/* Subtable recovery: each round iterates the r subtables        */
/* serially; subtable j's step snapshots its pure cells, recovers the set of  */
/* their keys and deletes each from all r cells, so later subtables of the    */
/* same round see those deletions.  Stops after a full round recovering       */
/* nothing.  *subrounds = flattened index (i-1) r + j of the last step that   */
/* recovered a key; per_sub[s-1] = keys recovered in flattened step s.        */
int ora_iblt_peel_subtables(ora_iblt *t, uint64_t *out_keys, uint64_t cap_keys, uint64_t *nrecovered,
                            uint32_t *subrounds, uint64_t *per_sub, uint32_t cap, int *complete) {
    if (!t->subtables) return -1;
    uint64_t C = t->C, cs = C / t->r;
    uint64_t *X = (uint64_t *)malloc(cs * sizeof(uint64_t));
    if (!X) return -1;
    uint64_t nrec = 0, flat = 0, last = 0;
    int status = 0;
    for (;;) {
        int any = 0;
        if (flat + t->r > ORA_IBLT_ROUND_LIMIT) { status = 1; break; }
        for (uint32_t j = 0; j < t->r; j++) {
            flat++;
            uint64_t nX = 0;
            for (uint64_t c = j * cs; c < (j + 1) * cs; c++)
                if (iblt_pure(t, c)) X[nX++] = t->keySum[c];
            qsort(X, nX, sizeof(uint64_t), cmp_u64);
            uint64_t u = 0;
            for (uint64_t i = 0; i < nX; i++)
                if (i == 0 || X[i] != X[i - 1]) X[u++] = X[i];
            nX = u;
            for (uint64_t i = 0; i < nX; i++) {
                iblt_apply(t, X[i], -1);
                if (nrec < cap_keys) out_keys[nrec] = X[i]; else status = 1;
                nrec++;
            }
            if (nX) { any = 1; last = flat; }
            if (flat <= cap) per_sub[flat - 1] = nX;
            else if (nX) status = 1;
        }
        if (!any) break;
    }
    free(X);
    *nrecovered = nrec;
    *subrounds = (uint32_t)last;
    int z = 1;
    for (uint64_t c = 0; c < C; c++)
        if (t->count[c] != 0 || t->keySum[c] != 0 || t->hashSum[c] != 0) { z = 0; break; }
    *complete = z;
    return status;
}

/* Set difference: a <- a - b cell-wise (count      */
/* subtracts, key and checksum fields XOR), the IBLT of the signed multiset   */
/* A - B.  Both tables must share C, r and seed.                              */
int ora_iblt_subtract(ora_iblt *a, const ora_iblt *b) {
    if (a->C != b->C || a->r != b->r || a->seed_h != b->seed_h || a->subtables != b->subtables || a->blog != b->blog)
        return -1;
    for (uint64_t c = 0; c < a->C; c++) {
        a->count[c] -= b->count[c];
        a->keySum[c] ^= b->keySum[c];
        a->hashSum[c] ^= b->hashSum[c];
    }
    return 0;
}

/* Round-synchronous recovery of a signed table: a cell is pure when its     */
/* count is +1 or -1, its checksum field equals checkSum(key field) and it is */
/* one of that key's cells (R26, R28).  Each round recovers every distinct    */
/* key x of the round-start pure cells ONCE, with the sign of the lowest-     */
/* index round-start pure cell holding x (R28), and removes it (deleting a +1 */
/* key, re-inserting a -1 key).  out_sign[i] is +1 for keys of A \ B, -1 for */
/* keys of B \ A.                                                           */
static int iblt_pure_signed(const ora_iblt *t, uint64_t c, int *sign) {
    if ((t->count[c] == 1 || t->count[c] == -1) && t->hashSum[c] == ora_checksum(t->keySum[c], t->seed_c) &&
        cell_of_key(t, c, t->keySum[c])) {
        *sign = (int)t->count[c];
        return 1;
    }
    return 0;
}

/* (key, cell, sign + 1) triples ordered by key, then cell */
static int cmp_key_cell(const void *a, const void *b) {
    const uint64_t *x = (const uint64_t *)a, *y = (const uint64_t *)b;
    if (x[0] != y[0]) return (x[0] > y[0]) - (x[0] < y[0]);
    return (x[1] > y[1]) - (x[1] < y[1]);
}

int ora_iblt_peel_signed(ora_iblt *t, uint64_t *out_keys, int8_t *out_sign, uint64_t cap_keys,
                         uint64_t *nrecovered, uint32_t *rounds, uint64_t *per_round, uint32_t cap,
                         int *complete) {
    uint64_t C = t->C;
    uint64_t *X = (uint64_t *)malloc(3 * C * sizeof(uint64_t));  /* (key, cell, sign + 1) */
    if (!X) return -1;
    uint64_t nrec = 0;
    uint32_t rt = 0;
    int status = 0;
    for (;;) {
        uint64_t nX = 0;
        for (uint64_t c = 0; c < C; c++) {
            int sg;
            if (iblt_pure_signed(t, c, &sg)) {
                X[3 * nX] = t->keySum[c]; X[3 * nX + 1] = c; X[3 * nX + 2] = (uint64_t)(sg + 1); nX++;
            }
        }
        if (nX == 0) break;
        if (rt == ORA_IBLT_ROUND_LIMIT) { status = 1; break; }
        qsort(X, nX, 3 * sizeof(uint64_t), cmp_key_cell);
        uint64_t u = 0;  /* first (lowest-cell) triple of every key */
        for (uint64_t i = 0; i < nX; i++)
            if (i == 0 || X[3 * i] != X[3 * (i - 1)]) {
                X[3 * u] = X[3 * i]; X[3 * u + 1] = X[3 * i + 1]; X[3 * u + 2] = X[3 * i + 2]; u++;
            }
        nX = u;
        rt += 1;
        for (uint64_t i = 0; i < nX; i++) {
            int sg = (int)X[3 * i + 2] - 1;
            iblt_apply(t, X[3 * i], -sg);
            if (nrec < cap_keys) { out_keys[nrec] = X[3 * i]; out_sign[nrec] = (int8_t)sg; } else status = 1;
            nrec++;
        }
        if (rt <= cap) per_round[rt - 1] = nX; else status = 1;
    }
    free(X);
    *nrecovered = nrec;
    *rounds = rt;
    int z = 1;
    for (uint64_t c = 0; c < C; c++)
        if (t->count[c] != 0 || t->keySum[c] != 0 || t->hashSum[c] != 0) { z = 0; break; }
    *complete = z;
    return status;
}

/* Serial recovery: repeatedly take ONE pure cell, recover its key,   */
/* delete it, until no pure cell remains.  A stack of candidate cells stands   */
/* in for "iteratively look for pure cells"; every cell is re-tested when     */
/* popped.  Recovered keys in recovery order.                                 */
int ora_iblt_serial_recover(ora_iblt *t, uint64_t *out_keys, uint64_t cap_keys,
                            uint64_t *nrecovered, int *complete) {
    uint64_t C = t->C;
    uint64_t cap_stack = C + 16 * C;
    uint64_t *stack = (uint64_t *)malloc(cap_stack * sizeof(uint64_t));
    if (!stack) return -1;
    uint64_t sp = 0, nrec = 0;
    int status = 0;
    for (uint64_t c = 0; c < C; c++) stack[sp++] = C - 1 - c;
    while (sp > 0) {
        uint64_t c = stack[--sp];
        if (!iblt_pure(t, c)) continue;
        uint64_t x = t->keySum[c];
        uint64_t cells[16];
        key_cells(t, x, cells);
        iblt_apply(t, x, -1);
        if (nrec < cap_keys) out_keys[nrec] = x; else status = 1;
        nrec++;
        for (uint32_t j = 0; j < t->r; j++)
            if (sp < cap_stack) stack[sp++] = cells[j];
    }
    free(stack);
    *nrecovered = nrec;
    int z = 1;
    for (uint64_t c = 0; c < C; c++)
        if (t->count[c] != 0 || t->keySum[c] != 0 || t->hashSum[c] != 0) { z = 0; break; }
    *complete = z;
    return status;
}

/* The IBLT's hypergraph: vertex = cell, edge = key's r cells.        */
void ora_iblt_to_hypergraph(const ora_iblt *t, const uint64_t *keys, uint64_t nkeys, uint32_t *edges) {
    uint64_t cells[16];
    for (uint64_t i = 0; i < nkeys; i++) {
        key_cells(t, keys[i], cells);
        for (uint32_t j = 0; j < t->r; j++) edges[i * t->r + j] = (uint32_t)cells[j];
    }
}
