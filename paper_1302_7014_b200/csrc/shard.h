// shard.h -- internal (not part of the C-ABI): the binned build of kcore.cu applied to one
// vertex shard [v0, v1) of an n-vertex instance, for the partitioned peel of dist.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "peel.h"

namespace peel {

// scratch bytes for shard_build (bin cursors, bases, capacities, flag, entries), or 0 if a
// shard of nloc vertices is small enough for the direct build (state <= 64 MB, L2-resident)
size_t shard_build_bytes(uint64_t n, uint64_t m, uint32_t r, uint64_t nloc);

// state[0 .. v1-v0) <- the packed (count | id sum << 32) states of the shard's vertices, from
// every edge of `edges` (validated: bad edges set ERR bit 1 in *err).  *overflow = true if a
// bin exceeded its capacity (adversarial degree skew): the caller then builds directly.
// Stream-ordered except for one small device-to-host read of the overflow flag.
// tmp / tmp_bytes: optional device scratch that is free during the build (dist.cu: the
// exchange buffers).  A narrow shard (v1 - v0 <= n / 4) with enough of it takes the filter
// path: one streaming pass keeps the shard's endpoints, a second bins them.
// f1 (optional): the build also scans the shard for F_1 while each bin is in L2 -- count < k
// adds to *nf, count-1 vertices append (v0 + i, id sum) to F at *ne (device counters, zeroed by
// the caller) -- and the caller skips its own scan.  Not done when *overflow comes back true.
struct ShardF1 {
    void *F;                   // uint2 [v1 - v0]
    unsigned long long *ne, *nf;
    uint32_t k;
};
peel_status shard_build(uint32_t r, const uint32_t *edges, uint64_t n, uint64_t m, uint64_t v0, uint64_t v1,
                        unsigned long long *state, uint32_t *err, char *scratch, cudaStream_t s, bool *overflow,
                        void *tmp = nullptr, size_t tmp_bytes = 0, const ShardF1 *f1 = nullptr);

// the shard's bins as the binned rounds use them: per-bin cursors and bases into `entries`
// (capacities from the build: a round's decrements of a bin are a subset of the build's),
// the apply phase's work counter, and an opaque control block for its counters
struct ShardBinsView {
    uint32_t nbins;
    unsigned long long *cursor;
    const unsigned long long *base;
    unsigned long long *entries;
    unsigned long long *work;
    char *ctl;
    unsigned long long *esort;  // edge-sort histogram and cursors
    uint32_t esort_words;       // their count (2 (edge bins + 1))
};
ShardBinsView shard_bins_view(uint64_t n, uint64_t m, uint32_t r, uint64_t nloc, char *scratch);

// phase D of a binned round t on the shard starting at vertex v0 (see kcore.cu)
peel_status shard_apply(uint64_t nloc, uint64_t v0, uint32_t k, unsigned long long *state, void *Fn,
                        const ShardBinsView &v, uint32_t t, unsigned long long *out_nf, unsigned long long *out_ne,
                        cudaStream_t s);

// the shard's frontier entries (v, e) [nE_host of them; *pN on the device] sorted by edge bin
// into dst (same capacity), as the single-GPU binned rounds do before their kill phase
// (zeroed: the caller has zeroed v.esort's 2 (enb + 1) counters on the stream already)
peel_status shard_edge_sort(const void *src, const unsigned long long *pN, uint64_t nE_host, uint64_t m, void *dst,
                            const ShardBinsView &v, cudaStream_t s, bool zeroed = false);

// BIN_SHIFT of kcore.cu (vertex bins of 2^22 local ids)
constexpr int SHARD_BIN_SHIFT = 22;

}  // namespace peel
