// iblt_common.cuh -- the IBLT cell and its hashes (R8, R25, R27),
// shared by the single-GPU table (iblt.cu) and the cell-partitioned table (iblt_dist.cu).
#pragma once
#include "common.cuh"

namespace peel {

struct __align__(16) Cell {
    uint32_t count;
    uint32_t hashSum;
    ull keySum;
};
static_assert(sizeof(Cell) == 16, "cell is 16 bytes");

// h_1(x)..h_r(x): r distinct cells
template <int R>
__device__ __forceinline__ void cells_of(ull x, ull C, ull seed_h, uint32_t (&c)[R]) {
    int na = 0;
    for (ull j = 0; na < R; j++) {
        ull z = mix64(x ^ seed_h ^ ((j + 1) * 0xD1B54A32D192ED03ull));
        uint32_t v = (uint32_t)__umul64hi(z, C);
        bool dup = false;
        #pragma unroll
        for (int i = 0; i < R; i++) dup |= (i < na) && (c[i] == v);
        if (!dup) {
            #pragma unroll
            for (int i = 0; i < R; i++) if (i == na) c[i] = v;
            na++;
        }
    }
}

// subtable hashing ("hash each item into one cell in each subtable"):
// h_j(x) = j C/r + umulhi64(mix64(x ^ seed_h ^ (j+1) 0xD1B54A32D192ED03), C/r)
// blocked hashing (IBLT_FLAG_BLOCKED; R27): block b = umulhi64(mix64(x ^ seed_h ^ K_B), C / B),
// then the plain r-distinct cells over B cells, offset by b B.  blog = 0: not blocked.
template <int R>
__device__ __forceinline__ void key_cells(ull x, ull C, ull seed_h, bool subt, uint32_t (&c)[R], uint32_t blog = 0) {
    if (blog) {
        const ull B = 1ull << blog;
        const ull b = __umul64hi(mix64(x ^ seed_h ^ 0x9E6C63D0676A9A99ull), C >> blog);
        cells_of<R>(x, B, seed_h, c);
        #pragma unroll
        for (int j = 0; j < R; j++) c[j] += (uint32_t)(b * B);
    } else if (subt) {
        const ull cs = C / R;
        #pragma unroll
        for (int j = 0; j < R; j++)
            c[j] = (uint32_t)(j * cs + __umul64hi(mix64(x ^ seed_h ^ ((ull)(j + 1) * 0xD1B54A32D192ED03ull)), cs));
    } else {
        cells_of<R>(x, C, seed_h, c);
    }
}

// checkSum(x)
__device__ __forceinline__ uint32_t checksum(ull x, ull seed_c) { return (uint32_t)(mix64(x ^ seed_c) >> 32); }

__device__ __forceinline__ Cell ld_cell_cg(const Cell *p) {
    uint4 v = __ldcg(reinterpret_cast<const uint4 *>(p));
    Cell c;
    c.count = v.x;
    c.hashSum = v.y;
    c.keySum = ((ull)v.w << 32) | v.z;
    return c;
}

__device__ __forceinline__ bool is_pure(const Cell &c, ull seed_c) {
    return c.count == 1u && c.hashSum == checksum(c.keySum, seed_c);
}

// DESIGN.md R28 ("cells that only contain one item"): a cell holding one item x is one
// of x's own cells, so purity also requires cell id c in h(keySum) -- a cell whose count and
// checksum say "pure" but whose key does not hash to it (a checksum collision, a forged or
// corrupted table) holds several items and is never recovered.  The hashes are computed only
// for cells that passed the count and checksum tests.
template <int R>
__device__ __forceinline__ bool cell_of_key(uint32_t c, ull x, ull C, ull seed_h, bool subt, uint32_t blog) {
    uint32_t h[R];
    key_cells<R>(x, C, seed_h, subt, h, blog);
    bool in = false;
    #pragma unroll
    for (int j = 0; j < R; j++) in |= h[j] == c;
    return in;
}

}  // namespace peel
