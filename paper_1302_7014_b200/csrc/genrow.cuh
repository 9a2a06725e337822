// genrow.cuh -- edge e of G^r_{n,.}(seed) as a pure function of (seed, n, r, e) (a1; P:89-91,
// P:363).  Shared by the generator kernels (gen.cu) and the sweep's per-trial groups (sweep.cu),
// which regenerate a killed edge's row instead of storing the edge list.  See gen.cu's header.
#pragma once
#include "common.cuh"

namespace peel {

// Philox4x32-10 (Salmon et al. SC'11), 10 rounds with Weyl key schedule.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    #pragma unroll
    for (int i = 0; i < 10; i++) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
}

// edge e of G^r_{n,.}(seed): r distinct vertices (see the header comment)
template <int R>
__device__ __forceinline__ void gen_one_edge(uint64_t e, uint64_t n, uint32_t k0, uint32_t k1, uint32_t (&acc)[R]) {
    int na = 0;
    uint32_t w[4];
    for (uint32_t j = 0; na < R; j++) {
        if ((j & 1) == 0) {
            w[0] = (uint32_t)e; w[1] = (uint32_t)(e >> 32); w[2] = j >> 1; w[3] = 0x45444745u;
            philox4x32_10(w, k0, k1);
        }
        uint64_t d = (j & 1) ? (((uint64_t)w[3] << 32) | w[2]) : (((uint64_t)w[1] << 32) | w[0]);
        uint32_t v = (uint32_t)__umul64hi(d, n);
        bool dup = false;
        #pragma unroll
        for (int i = 0; i < R; i++) dup |= (i < na) && (acc[i] == v);
        if (!dup) {
            #pragma unroll
            for (int i = 0; i < R; i++) if (i == na) acc[i] = v;
            na++;
        }
    }
}

}  // namespace peel
