// gen.cu -- a1: counter-based generator of G^r_{n,cn} edges and IBLT keys.
//
// P:89-91 / P:363: m independent hyperedges, each r DISTINCT vertices chosen
// uniformly.  Edge e is a pure function of (seed, n, r, e), so one thread per
// edge needs no coordination: draw j = half (j%2) of Philox4x32-10 block
// (ctr = {e_lo, e_hi, j/2, 'EDGE'}, key = {seed_lo, seed_hi}); vertex =
// umulhi64(draw, n); rejected if already in the edge.
#include "common.cuh"
#include "genrow.cuh"

namespace peel {

template <int R>
__global__ void __launch_bounds__(256) gen_edges_kernel(uint64_t n, uint64_t m, uint64_t seed,
                                                        uint32_t *__restrict__ edges, uint32_t voff) {
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t acc[R];
        gen_one_edge<R>(e, n, k0, k1, acc);
        #pragma unroll
        for (int i = 0; i < R; i++) edges[e * R + i] = acc[i] + voff;
    }
}

// a batch of B trials in one launch (peel_sweep): edge g of the concatenation belongs to
// trial b with mpre[b] <= g < mpre[b+1]; it is edge g - mpre[b] of G^r_{n,m_b}(seeds[b])
// with every vertex shifted by b n -- the same edges as B gen_edges_kernel launches.
static constexpr int GB_MAX = 1024;

template <int R>
__global__ void __launch_bounds__(256) gen_batch_kernel(uint64_t n, uint32_t B, const uint64_t *__restrict__ mpre,
                                                        const uint64_t *__restrict__ seeds, uint32_t *__restrict__ edges) {
    __shared__ uint64_t sp[GB_MAX + 1];
    for (uint32_t i = threadIdx.x; i <= B; i += 256) sp[i] = mpre[i];
    __syncthreads();
    const uint64_t total = sp[B];
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = B;  // trial b: sp[b] <= g < sp[b+1]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (sp[mid] <= g) lo = mid; else hi = mid;
        }
        const uint64_t seed = seeds[lo];
        uint32_t acc[R];
        gen_one_edge<R>(g - sp[lo], n, (uint32_t)seed, (uint32_t)(seed >> 32), acc);
        const uint32_t voff = (uint32_t)(lo * n);
        #pragma unroll
        for (int i = 0; i < R; i++) edges[g * R + i] = acc[i] + voff;
    }
}

// the subtable model: one uniform vertex per class, draw c for class c
template <int R>
__global__ void __launch_bounds__(256) gen_partitioned_kernel(uint64_t m, uint64_t cs, uint64_t seed,
                                                              uint32_t *__restrict__ edges) {
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t w[4];
        #pragma unroll
        for (int c = 0; c < R; c++) {
            if ((c & 1) == 0) {
                w[0] = (uint32_t)e; w[1] = (uint32_t)(e >> 32); w[2] = (uint32_t)c >> 1; w[3] = 0x53554254u;
                philox4x32_10(w, k0, k1);
            }
            const uint64_t d = (c & 1) ? (((uint64_t)w[3] << 32) | w[2]) : (((uint64_t)w[1] << 32) | w[0]);
            edges[e * R + c] = (uint32_t)(c * cs + __umul64hi(d, cs));
        }
    }
}

__global__ void __launch_bounds__(256) gen_keys_kernel(uint64_t nkeys, uint64_t seed,
                                                       uint64_t *__restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nkeys;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
}

static unsigned grid_for(uint64_t work, int per_sm = 16) {
    uint64_t blocks = (work + 255) / 256;
    uint64_t cap = (uint64_t)num_sms() * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    return (unsigned)blocks;
}

}  // namespace peel

using namespace peel;

namespace peel {
// edges[m][r] of G^r_{n,cn}(seed) with every vertex id shifted by voff (voff = 0: the ABI call;
// voff = b n: trial b of a disjoint-union batch, peel_sweep)
peel_status launch_gen_edges(uint64_t n, uint64_t m, uint32_t r, uint64_t seed, uint32_t *edges, uint32_t voff,
                             cudaStream_t s) {
    unsigned g = grid_for(m);
    ProfScope ps("gen_edges", s);
    switch (r) {
        case 2: gen_edges_kernel<2><<<g, 256, 0, s>>>(n, m, seed, edges, voff); break;
        case 3: gen_edges_kernel<3><<<g, 256, 0, s>>>(n, m, seed, edges, voff); break;
        case 4: gen_edges_kernel<4><<<g, 256, 0, s>>>(n, m, seed, edges, voff); break;
        case 5: gen_edges_kernel<5><<<g, 256, 0, s>>>(n, m, seed, edges, voff); break;
        case 6: gen_edges_kernel<6><<<g, 256, 0, s>>>(n, m, seed, edges, voff); break;
        case 7: gen_edges_kernel<7><<<g, 256, 0, s>>>(n, m, seed, edges, voff); break;
        case 8: gen_edges_kernel<8><<<g, 256, 0, s>>>(n, m, seed, edges, voff); break;
        default: return PEEL_EINVAL;
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}
}  // namespace peel

namespace peel {
// the B trials' edges, concatenated (mpre: B+1 prefix sums of m, device; seeds: B, device)
peel_status launch_gen_batch(uint64_t n, uint32_t r, uint32_t B, const uint64_t *mpre, const uint64_t *seeds,
                             uint64_t total, uint32_t *edges, cudaStream_t s) {
    if (B > GB_MAX) return PEEL_EINVAL;
    if (total == 0) return PEEL_OK;
    unsigned g = grid_for(total);
    ProfScope ps("gen_edges_batch", s);
    switch (r) {
        case 2: gen_batch_kernel<2><<<g, 256, 0, s>>>(n, B, mpre, seeds, edges); break;
        case 3: gen_batch_kernel<3><<<g, 256, 0, s>>>(n, B, mpre, seeds, edges); break;
        case 4: gen_batch_kernel<4><<<g, 256, 0, s>>>(n, B, mpre, seeds, edges); break;
        case 5: gen_batch_kernel<5><<<g, 256, 0, s>>>(n, B, mpre, seeds, edges); break;
        case 6: gen_batch_kernel<6><<<g, 256, 0, s>>>(n, B, mpre, seeds, edges); break;
        case 7: gen_batch_kernel<7><<<g, 256, 0, s>>>(n, B, mpre, seeds, edges); break;
        case 8: gen_batch_kernel<8><<<g, 256, 0, s>>>(n, B, mpre, seeds, edges); break;
        default: return PEEL_EINVAL;
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}
}  // namespace peel

extern "C" peel_status peel_gen_hypergraph(uint64_t n, uint64_t m, uint32_t r, uint64_t seed,
                                           uint32_t *edges, void *stream) {
    if (r < 2 || r > 8 || n < r || n > (1ull << 32) || m >= (1ull << 32)) return PEEL_EINVAL;
    if (m == 0) return PEEL_OK;
    if (!edges) return PEEL_EINVAL;
    prof_begin_call();
    return launch_gen_edges(n, m, r, seed, edges, 0u, (cudaStream_t)stream);
}

extern "C" peel_status peel_gen_partitioned(uint64_t n, uint64_t m, uint32_t r, uint64_t seed, uint32_t *edges,
                                            void *stream) {
    if (r < 2 || r > 8 || n < r || n % r || n > (1ull << 32) || m >= (1ull << 32)) return PEEL_EINVAL;
    if (m == 0) return PEEL_OK;
    if (!edges) return PEEL_EINVAL;
    prof_begin_call();
    cudaStream_t s = (cudaStream_t)stream;
    const uint64_t cs = n / r;
    unsigned g = grid_for(m);
    {
        ProfScope ps("gen_partitioned", s);
        switch (r) {
            case 2: gen_partitioned_kernel<2><<<g, 256, 0, s>>>(m, cs, seed, edges); break;
            case 3: gen_partitioned_kernel<3><<<g, 256, 0, s>>>(m, cs, seed, edges); break;
            case 4: gen_partitioned_kernel<4><<<g, 256, 0, s>>>(m, cs, seed, edges); break;
            case 5: gen_partitioned_kernel<5><<<g, 256, 0, s>>>(m, cs, seed, edges); break;
            case 6: gen_partitioned_kernel<6><<<g, 256, 0, s>>>(m, cs, seed, edges); break;
            case 7: gen_partitioned_kernel<7><<<g, 256, 0, s>>>(m, cs, seed, edges); break;
            case 8: gen_partitioned_kernel<8><<<g, 256, 0, s>>>(m, cs, seed, edges); break;
        }
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}

extern "C" peel_status peel_gen_keys(uint64_t nkeys, uint64_t seed, uint64_t *keys, void *stream) {
    if (nkeys == 0) return PEEL_OK;
    if (!keys) return PEEL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    prof_begin_call();
    {
        ProfScope ps("gen_keys", s);
        gen_keys_kernel<<<grid_for(nkeys), 256, 0, s>>>(nkeys, seed, keys);
    }
    PEEL_CUDA(cudaGetLastError());
    return PEEL_OK;
}
