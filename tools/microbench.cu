// microbench.cu — B200 rates that decide the histogram / ranking designs:
// shared-memory atomics (random bins, with and without return), match.any,
// global RED, and the L2 round trip of ld.relaxed.gpu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <int MODE>  // 0 atomicAdd no-ret 32-bit, 1 with return, 2 packed 16-bit with return
__global__ void k_smem_atomic(uint32_t iters, uint32_t mask, uint32_t *out)
{
    extern __shared__ uint32_t sh[];
    const uint32_t words = MODE == 2 ? (mask + 1) / 2 : mask + 1;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    uint32_t seed = hash32(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    for (uint32_t it = 0; it < iters; it++) {
        uint32_t b = hash32(seed + it * 0x9e3779b9u) & mask;
        if (MODE == 0) atomicAdd(&sh[b], 1u);
        else if (MODE == 1) acc += atomicAdd(&sh[b], 1u);
        else acc += atomicAdd(&sh[b >> 1], 1u << ((b & 1) << 4));
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sh[0] + acc;
}

__global__ void k_match(uint32_t iters, uint32_t mask, uint32_t *out)
{
    uint32_t seed = hash32(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    for (uint32_t it = 0; it < iters; it++) {
        uint32_t b = hash32(seed + it * 0x9e3779b9u) & mask;
        acc += __match_any_sync(0xffffffffu, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_hashonly(uint32_t iters, uint32_t mask, uint32_t *out)
{
    uint32_t seed = hash32(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    for (uint32_t it = 0; it < iters; it++) acc += hash32(seed + it * 0x9e3779b9u) & mask;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_gred(uint32_t iters, uint32_t mask, uint32_t *g)
{
    uint32_t seed = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (uint32_t it = 0; it < iters; it++) atomicAdd(&g[hash32(seed + it * 0x9e3779b9u) & mask], 1u);
}

__global__ void k_chase(const uint32_t *p, uint32_t iters, uint32_t *out)
{
    uint32_t j = 0;
    for (uint32_t i = 0; i < iters; i++) {
        uint32_t v;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p + j) : "memory");
        j = v;
    }
    out[0] = j;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out, *g;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&g, 1 << 22);
    cudaMemset(g, 0, 1 << 22);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    const uint32_t iters = 4096;
    cudaFuncSetAttribute(k_smem_atomic<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    cudaFuncSetAttribute(k_smem_atomic<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    cudaFuncSetAttribute(k_smem_atomic<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    for (int threads : {256, 1024}) {
        for (uint32_t bins : {256u, 4096u, 32768u, 65536u}) {
            for (int mode = 0; mode < 3; mode++) {
                size_t smem = (mode == 2 ? bins / 2 : bins) * 4;
                if (mode == 2 && bins < 512) continue;
                if (smem > 140 * 1024) continue;
                int ctas = sms * (threads == 256 ? 4 : 1);
                if (smem * (threads == 256 ? 4 : 1) > 200 * 1024) ctas = sms;
                auto run = [&] {
                    if (mode == 0) k_smem_atomic<0><<<ctas, threads, smem>>>(iters, bins - 1, out);
                    if (mode == 1) k_smem_atomic<1><<<ctas, threads, smem>>>(iters, bins - 1, out);
                    if (mode == 2) k_smem_atomic<2><<<ctas, threads, smem>>>(iters, bins - 1, out);
                };
                run();
                cudaEventRecord(a);
                run();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                if (cudaGetLastError() != cudaSuccess) { printf("error\n"); return 1; }
                cudaEventElapsedTime(&ms, a, b);
                double ops = (double)ctas * threads * iters;
                printf("smem_atomic mode=%d threads=%d ctas=%d bins=%u: %.1f Gatom/s  %.2f atom/clk/SM@1.9GHz\n",
                       mode, threads, ctas, bins, ops / ms / 1e6, ops / ms / 1e6 / sms / 1.9);
            }
        }
    }
    for (uint32_t mask : {15u, 255u, 65535u}) {
        int ctas = sms * 4, threads = 256;
        k_match<<<ctas, threads>>>(iters, mask, out);
        cudaEventRecord(a);
        k_match<<<ctas, threads>>>(iters, mask, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)ctas * threads * iters;
        float ms2;
        k_hashonly<<<ctas, threads>>>(iters, mask, out);
        cudaEventRecord(a);
        k_hashonly<<<ctas, threads>>>(iters, mask, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms2, a, b);
        printf("match_any mask=%u: %.1f Glane/s (%.2f lane/clk/SM), hash-only %.1f Glane/s\n", mask,
               ops / ms / 1e6, ops / ms / 1e6 / sms / 1.9, ops / ms2 / 1e6);
    }
    for (uint32_t mask : {65535u, (1u << 20) - 1}) {
        int ctas = sms * 4, threads = 256;
        uint32_t it2 = 256;
        k_gred<<<ctas, threads>>>(it2, mask, g);
        cudaEventRecord(a);
        k_gred<<<ctas, threads>>>(it2, mask, g);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)ctas * threads * it2;
        printf("global RED random over %u words: %.1f Gatom/s\n", mask + 1, ops / ms / 1e6);
    }
    // L2 round trip: pointer chase over a 1 MiB ring with a 4 KiB stride
    {
        const int N = 1 << 18;
        uint32_t *h = new uint32_t[N];
        for (int i = 0; i < N; i++) h[i] = (i + 1024 + 7) % N;
        uint32_t *d;
        cudaMalloc(&d, N * 4);
        cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
        k_chase<<<1, 1>>>(d, 1000, out);
        cudaEventRecord(a);
        k_chase<<<1, 1>>>(d, 20000, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("ld.relaxed.gpu L2 round trip: %.1f ns\n", ms * 1e6 / 20000);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
