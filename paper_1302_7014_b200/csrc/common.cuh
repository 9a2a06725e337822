// common.cuh -- shared device/host helpers of libpeel (product path; no oracle code).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "peel.h"

namespace cg = cooperative_groups;

namespace peel {

typedef unsigned long long ull;

// ---------------------------------------------------------------------------
// host-side error plumbing
// ---------------------------------------------------------------------------
void set_cuda_error(cudaError_t e, const char *where);

#define PEEL_CUDA(call)                                   \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) {                          \
            ::peel::set_cuda_error(_e, #call);            \
            return PEEL_ECUDA;                            \
        }                                                 \
    } while (0)

// ---------------------------------------------------------------------------
// per-call launch accounting + optional CUDA-event profiling (peel.h)
// ---------------------------------------------------------------------------
void prof_begin_call();                                   // resets the per-call tables
int prof_pre(const char *name, cudaStream_t s);           // before a kernel launch: its entry, or -1
void prof_post(int entry, cudaStream_t s);                // after it (counts the launch)
int prof_collect();                                       // after stream sync: resolve events
bool prof_enabled();
void prof_hold(bool on);  // nest public calls inside one report (peel_sweep)
void prof_add_launches(uint32_t n);  // kernels launched inside a replayed CUDA graph
void prof_capture(bool on);          // suppress profiling while a stream is being captured
void prof_set_rounds(const std::vector<double> &ms);      // per-round device time of the last peel

struct ProfScope {
    const char *name;
    cudaStream_t s;
    int entry;
    ProfScope(const char *n, cudaStream_t st) : name(n), s(st) { entry = prof_pre(n, st); }
    ~ProfScope() { prof_post(entry, s); }
};

// number of SMs and cooperative occupancy helpers
int num_sms();

// raise (never lower) a kernel's dynamic shared-memory limit on the current device: host threads
// calling the library concurrently with different sizes must not lower another's launch limit
cudaError_t raise_smem(const void *kern, size_t bytes);

// generator launch shared by peel_gen_hypergraph and peel_sweep (gen.cu)
peel_status launch_gen_edges(uint64_t n, uint64_t m, uint32_t r, uint64_t seed, uint32_t *edges, uint32_t voff,
                             cudaStream_t s);
peel_status launch_gen_batch(uint64_t n, uint32_t r, uint32_t B, const uint64_t *mpre, const uint64_t *seeds,
                             uint64_t total, uint32_t *edges, cudaStream_t s);

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ ull ld_cg_u64(const ull *p) { return __ldcg(p); }

// acquire load (gpu scope): spin-waits on counters other blocks release with a fence + atomic
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// bulk prefetch of [p, p + bytes) into L2 (p and bytes multiples of 16)
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// prefetch the L2 line holding p (fire and forget)
__device__ __forceinline__ void prefetch_line_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// %globaltimer (ns): per-round device timestamps for profiling
__device__ __forceinline__ ull globaltimer() {
    ull t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The R vertex ids of edge e, read with the 16-byte vector loads that cover the row
// (R = 3: two 8-byte loads; R = 2, 4: one load) instead of R scalar loads: measured with
// ncu, the scalar loads of one random row reach L2 as separate requests and miss separately
// (DRAM reads 2x the rows' granules).  vec: edges is 16-byte aligned; m R words in total.
template <int R>
__device__ __forceinline__ void load_row(const uint32_t *__restrict__ edges, uint64_t e, uint64_t m, bool vec,
                                         uint32_t (&u)[R]) {
    const uint64_t w0 = e * R;
    const uint64_t end = m * R;  // words in the array
    if (R == 3 && vec && (w0 | 1) + 3 <= end) {  // two 8-byte loads, branch-free
        const uint2 *p2 = reinterpret_cast<const uint2 *>(edges) + (w0 >> 1);
        const uint2 x = __ldg(p2), y = __ldg(p2 + 1);
        const bool odd = (w0 & 1) != 0;
        u[0] = odd ? x.y : x.x;
        u[1 % R] = odd ? y.x : x.y;
        u[2 % R] = odd ? y.y : y.x;
        return;
    }
    if (R == 2 && vec) {  // rows are 8-byte aligned
        const uint2 x = __ldg(reinterpret_cast<const uint2 *>(edges) + (w0 >> 1));
        u[0] = x.x;
        u[1 % R] = x.y;
        return;
    }
    const uint64_t q0 = w0 >> 2, q1 = (w0 + R - 1) >> 2;  // first / last 16-byte window
    if (R <= 3 || !vec || (q1 + 1) * 4 > end) {             // unaligned array, or a window past its end
        #pragma unroll
        for (int j = 0; j < R; j++) u[j] = __ldg(edges + w0 + j);
        return;
    }
    constexpr int NQ = (R + 6) / 4;  // windows a row can span
    uint32_t w[4 * NQ];
    const uint4 *p = reinterpret_cast<const uint4 *>(edges);
    #pragma unroll
    for (int i = 0; i < NQ; i++) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (i == 0 || q0 + i <= q1) v = __ldg(p + q0 + i);
        w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
    switch ((uint32_t)(w0 & 3)) {  // constant register indices in every case
        case 0:
            #pragma unroll
            for (int j = 0; j < R; j++) u[j] = w[j];
            break;
        case 1:
            #pragma unroll
            for (int j = 0; j < R; j++) u[j] = w[j + 1];
            break;
        case 2:
            #pragma unroll
            for (int j = 0; j < R; j++) u[j] = w[j + 2];
            break;
        default:
            #pragma unroll
            for (int j = 0; j < R; j++) u[j] = w[j + 3];
            break;
    }
}
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t *p) { return __ldcg(p); }

// SplitMix64 finalizer (Steele-Lea-Flood); the IBLT hash/checksum mixer.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Warp-aggregated append of `v` to list[counter++] for the threads that call
// it (all calling threads must be converged at the call, e.g. inside `if`).
template <typename T>
__device__ __forceinline__ ull append(T *list, ull *counter, T v) {
    cg::coalesced_group g = cg::coalesced_threads();
    ull base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(counter, (ull)g.size());
    base = g.shfl(base, 0);
    list[base + g.thread_rank()] = v;
    return base + g.thread_rank();
}

// block-wide sum of a per-thread u64, one atomicAdd per block into *dst.
template <int BLOCK>
__device__ __forceinline__ void block_add(ull *dst, ull v) {
    __shared__ ull red[BLOCK / 32];
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < BLOCK / 32 ? red[lane] : 0;
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(dst, v);
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Block-aggregated append queue (double-buffered in shared memory).
// Threads push with one shared-memory atomic per warp; at the end of every
// block-uniform iteration the block reserves space in the global list with ONE
// global atomic and copies the batch out coalesced.  A single global counter hit
// by every warp serialises at one L2 slice (measured ~1.5e9 atomics/s on B200:
// 0.5 s on the 10^9-vertex instance before this).  Iteration i pushes into slot
// i&1, so the copy-out of slot i&1 never races with the next iteration's pushes.
// Overflow beyond QCAP falls back to a warp-aggregated global append, so
// correctness never depends on QCAP.
// ---------------------------------------------------------------------------
template <typename T, int QCAP, int BLOCK>
struct BlockQueueT {
    T buf[2][QCAP];
    uint32_t n[2];
    uint32_t cnt;
    ull base;
};

template <typename T, int QCAP, int BLOCK>
__device__ __forceinline__ void bq_init(BlockQueueT<T, QCAP, BLOCK> &q) {
    if (threadIdx.x == 0) { q.n[0] = 0; q.n[1] = 0; }
}

// NOTE: warp-aggregated -- every thread of the coalesced group at the call site must
// push to the SAME queue q (call it under a warp-uniform selection of q).
template <typename T, int QCAP, int BLOCK>
__device__ __forceinline__ void bq_push(BlockQueueT<T, QCAP, BLOCK> &q, int slot, T v, T *gl, ull *gcnt) {
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t pos = 0;
    if (g.thread_rank() == 0) pos = atomicAdd(&q.n[slot], (uint32_t)g.size());
    pos = g.shfl(pos, 0) + g.thread_rank();
    if (pos < QCAP) {
        q.buf[slot][pos] = v;
    } else {
        cg::coalesced_group h = cg::coalesced_threads();
        ull b = 0;
        if (h.thread_rank() == 0) b = atomicAdd(gcnt, (ull)h.size());
        gl[h.shfl(b, 0) + h.thread_rank()] = v;
    }
}

// every thread of the block must call it.  Entries at positions >= cap of the
// global list are counted but not stored (callers with bounded outputs).
template <typename T, int QCAP, int BLOCK>
__device__ __forceinline__ void bq_flush(BlockQueueT<T, QCAP, BLOCK> &q, int slot, T *gl, ull *gcnt,
                                         ull cap = ~0ull) {
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = min(q.n[slot], (uint32_t)QCAP);
        q.cnt = c;
        q.base = c ? atomicAdd(gcnt, (ull)c) : 0ull;
        q.n[slot] = 0;
    }
    __syncthreads();
    const uint32_t c = q.cnt;
    const ull b = q.base;
    for (uint32_t i = threadIdx.x; i < c; i += BLOCK)
        if (b + i < cap) gl[b + i] = q.buf[slot][i];
}

// bq_flush with a custom writer: writer(global_index, value) for each queued value
// (e.g. to split a queued pair into two output arrays).  Same contract as bq_flush.
template <typename T, int QCAP, int BLOCK, typename W>
__device__ __forceinline__ void bq_flush_with(BlockQueueT<T, QCAP, BLOCK> &q, int slot, ull *gcnt, ull cap, W writer) {
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = min(q.n[slot], (uint32_t)QCAP);
        q.cnt = c;
        q.base = c ? atomicAdd(gcnt, (ull)c) : 0ull;
        q.n[slot] = 0;
    }
    __syncthreads();
    const uint32_t c = q.cnt;
    const ull b = q.base;
    for (uint32_t i = threadIdx.x; i < c; i += BLOCK)
        if (b + i < cap) writer(b + i, q.buf[slot][i]);
}

}  // namespace peel
