// membench.cu -- B200 microbenchmarks that decide the peel's memory design
// (SURVEY §7 "measure first"): random gather / RED / ATOM rates vs working-set
// size, L2-resident atomics, shared-memory atomics, single-address contention.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

typedef unsigned long long ull;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ ull hash64(ull z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_copy(const ull *__restrict__ a, ull *__restrict__ b, ull n) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_gather(const ull *__restrict__ a, ull span, ull nops, ull *out) {
    ull acc = 0;
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x)
        acc += __ldcg(a + (hash64(i) % span));
    if (acc == 12345) out[0] = acc;
}
__global__ void k_gather16(const uint4 *__restrict__ a, ull span, ull nops, ull *out) {
    unsigned acc = 0;
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x) {
        uint4 v = __ldcg(a + (hash64(i) % span));
        acc += v.x ^ v.w;
    }
    if (acc == 12345) out[0] = acc;
}
__global__ void k_red(ull *a, ull span, ull nops) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x)
        atomicAdd(a + (hash64(i) % span), 1ull);
}
__global__ void k_atom(ull *a, ull span, ull nops, ull *out) {
    ull acc = 0;
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x)
        acc += atomicAdd(a + (hash64(i) % span), 1ull);
    if (acc == 12345) out[0] = acc;
}
__global__ void k_red32(unsigned *a, ull span, ull nops) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x)
        atomicAdd(a + (hash64(i) % span), 1u);
}
__global__ void k_and32(unsigned *a, ull span, ull nops, ull *out) {
    unsigned acc = 0;
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x) {
        ull h = hash64(i);
        acc ^= atomicAnd(a + (h % span), ~(1u << (h >> 59)));
    }
    if (acc == 12345) out[0] = acc;
}
// shared-memory RED.u64 into a 24K-entry table per block
__global__ void k_smem_red(ull nops_per_block, ull *out) {
    extern __shared__ ull tab[];
    const int N = 24576;
    for (int i = threadIdx.x; i < N; i += blockDim.x) tab[i] = 0;
    __syncthreads();
    for (ull i = threadIdx.x; i < nops_per_block; i += blockDim.x)
        atomicAdd(tab + (hash64(i ^ ((ull)blockIdx.x << 40)) % N), 1ull);
    __syncthreads();
    if (tab[threadIdx.x] == 12345) out[0] = 1;
}
__global__ void k_single(ull *c, ull nops) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x)
        atomicAdd(c, 1ull);
}
// random 8B store (scatter) into a large array
__global__ void k_scatter(ull *a, ull span, ull nops) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x)
        a[hash64(i) % span] = i;
}
// "binned" scatter: writes go to B bins with per-warp cursors (append), 8B entries
__global__ void k_binned_append(ull *buf, ull bin_cap, unsigned nbins, ull *cursors, ull nops) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < nops; i += (ull)gridDim.x * blockDim.x) {
        ull h = hash64(i);
        unsigned b = (unsigned)(h % nbins);
        ull pos = atomicAdd(cursors + b * 16, 1ull);
        if (pos < bin_cap) buf[(ull)b * bin_cap + pos] = h;
    }
}

static float timeit(void (*launch)(void *), void *ctx, int reps = 3) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    launch(ctx);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; r++) {
        cudaEventRecord(a);
        launch(ctx);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

struct Ctx { ull *a, *b, *out; ull span, nops; int grid, block; unsigned nb; ull cap; };
static Ctx C;
static int SMS;

int main() {
    int dev = 0;
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
    SMS = p.multiProcessorCount;
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d}\n", p.name, SMS, p.l2CacheSize, p.clockRate);
    const ull BIG = 1ull << 30;  // 1G u64 = 8 GiB
    CK(cudaMalloc(&C.a, BIG * 8));
    CK(cudaMalloc(&C.b, BIG * 8 + 4096));
    CK(cudaMalloc(&C.out, 4096));
    CK(cudaMemset(C.a, 0, BIG * 8));
    C.grid = SMS * 8; C.block = 256;
    const ull NOPS = 1ull << 28;  // 268M ops

    float ms = timeit([](void *) { k_copy<<<C.grid, C.block>>>(C.a, C.b, 1ull << 30); }, 0);
    printf("{\"test\": \"seq_copy_8GiB\", \"ms\": %.3f, \"GBps\": %.1f}\n", ms, 2.0 * 8 * (1ull << 30) / ms / 1e6);

    {
        size_t g0 = 0;
        cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity);
        printf("{\"l2_fetch_granularity_default\": %zu}\n", g0);
        for (size_t gran : {32, 64, 128}) {
            cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
            size_t got = 0;
            cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
            C.span = 1ull << 30; C.nops = NOPS;
            float g = timeit([](void *) { k_gather<<<C.grid, C.block>>>(C.a, C.span, C.nops, C.out); }, 0);
            float r = timeit([](void *) { k_red<<<C.grid, C.block>>>(C.a, C.span, C.nops); }, 0);
            float t = timeit([](void *) { k_atom<<<C.grid, C.block>>>(C.a, C.span, C.nops, C.out); }, 0);
            printf("{\"test\": \"random_u64_8GiB_fetch_gran\", \"set\": %zu, \"got\": %zu, \"err\": %d, \"gather_Gops\": %.2f, \"red_Gops\": %.2f, \"atom_Gops\": %.2f}\n",
                   gran, got, (int)e, NOPS / g / 1e6, NOPS / r / 1e6, NOPS / t / 1e6);
        }
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g0);
    }
    ull spans[] = {1ull << 30, 1ull << 27, 1ull << 25, 1ull << 23, 1ull << 21, 1ull << 18};
    for (ull sp : spans) {
        C.span = sp; C.nops = NOPS;
        float g = timeit([](void *) { k_gather<<<C.grid, C.block>>>(C.a, C.span, C.nops, C.out); }, 0);
        float r = timeit([](void *) { k_red<<<C.grid, C.block>>>(C.a, C.span, C.nops); }, 0);
        float t = timeit([](void *) { k_atom<<<C.grid, C.block>>>(C.a, C.span, C.nops, C.out); }, 0);
        float s = timeit([](void *) { k_scatter<<<C.grid, C.block>>>(C.b, C.span, C.nops); }, 0);
        printf("{\"test\": \"random_u64\", \"span_bytes\": %llu, \"gather_Gops\": %.2f, \"red_Gops\": %.2f, \"atom_Gops\": %.2f, \"scatter_Gops\": %.2f}\n",
               sp * 8, NOPS / g / 1e6, NOPS / r / 1e6, NOPS / t / 1e6, NOPS / s / 1e6);
    }
    for (ull sp : {1ull << 30, 1ull << 25}) {
        C.span = sp / 2; C.nops = NOPS;
        float g = timeit([](void *) { k_gather16<<<C.grid, C.block>>>((const uint4 *)C.a, C.span, C.nops, C.out); }, 0);
        printf("{\"test\": \"random_16B_gather\", \"span_bytes\": %llu, \"Gops\": %.2f}\n", sp * 8, NOPS / g / 1e6);
    }
    for (ull sp : {1ull << 31, 1ull << 25, 1ull << 22}) {  // u32 words
        C.span = sp; C.nops = NOPS;
        float r = timeit([](void *) { k_red32<<<C.grid, C.block>>>((unsigned *)C.a, C.span, C.nops); }, 0);
        float t = timeit([](void *) { k_and32<<<C.grid, C.block>>>((unsigned *)C.a, C.span, C.nops, C.out); }, 0);
        printf("{\"test\": \"random_u32\", \"span_bytes\": %llu, \"red32_Gops\": %.2f, \"atomand32_Gops\": %.2f}\n", sp * 4, NOPS / r / 1e6, NOPS / t / 1e6);
    }
    {
        CK(cudaFuncSetAttribute(k_smem_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 24576 * 8));
        C.nops = 1ull << 22;
        float ms2 = timeit([](void *) { k_smem_red<<<SMS, 1024, 24576 * 8>>>(C.nops, C.out); }, 0);
        printf("{\"test\": \"smem_red_u64\", \"Gops\": %.2f}\n", (double)SMS * C.nops / ms2 / 1e6);
    }
    {
        C.nops = 1ull << 24;
        float ms3 = timeit([](void *) { k_single<<<C.grid, C.block>>>(C.out, C.nops); }, 0);
        printf("{\"test\": \"single_address_atomic\", \"Gops\": %.3f}\n", C.nops / ms3 / 1e6);
    }
    for (unsigned nb : {256u, 4096u, 32768u}) {
        C.nb = nb; C.nops = NOPS; C.cap = (NOPS / nb) * 2;
        CK(cudaMemset(C.out, 0, 4096));
        ull *cur; CK(cudaMalloc(&cur, (ull)nb * 16 * 8));
        C.a = C.a;  // reuse
        static ull *curs; curs = cur;
        struct L { static void f(void *c) { k_binned_append<<<C.grid, C.block>>>(C.b, C.cap, C.nb, (ull *)c, C.nops); } };
        cudaMemset(cur, 0, (ull)nb * 16 * 8);
        float t = timeit([](void *c) { cudaMemset(c, 0, (ull)C.nb * 16 * 8); k_binned_append<<<C.grid, C.block>>>(C.b, C.cap, C.nb, (ull *)c, C.nops); }, cur);
        printf("{\"test\": \"binned_append_naive\", \"bins\": %u, \"Gops\": %.2f}\n", nb, NOPS / t / 1e6);
        cudaFree(cur);
    }
    return 0;
}
