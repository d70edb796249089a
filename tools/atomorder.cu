// atomorder.cu — does B200 serve same-address shared-memory atomics of one
// warp instruction in ascending lane order?  (The CUDA model leaves it
// unspecified; this only measures what the hardware does.)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ao tools/atomorder.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <int MODE>  // 0: add 1; 1: add (1<<16+lane%16)+1 as in the ranking word; 2: 64-bit add
__global__ void k_order(int iters, uint32_t nvals, unsigned long long *bad, unsigned long long *total)
{
    __shared__ uint32_t tab[32][256];
    __shared__ unsigned long long tab64[16][256];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) (&tab[0][0])[i] = 0;
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) (&tab64[0][0])[i] = 0;
    __syncthreads();
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    unsigned long long nbad = 0, ntot = 0;
    uint32_t seed = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (int it = 0; it < iters; it++) {
        const uint32_t r = hash32(seed + it * 0x9e3779b9u);
        const uint32_t d = (r % nvals) * (256 / nvals);  // spread values over the table
        uint32_t old;
        if (MODE == 0) old = atomicAdd(&tab[warp][d], 1u);
        else if (MODE == 1) old = atomicAdd(&tab[warp][d], (1u << (16 + (lane & 15))) + 1u) & 0xffffu;
        else old = (uint32_t)atomicAdd(&tab64[warp & 15][d], 1ull);
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t first = __ffs(peers) - 1;
        const uint32_t base = __shfl_sync(0xffffffffu, old, first);
        nbad += (old != base + __popc(peers & lt)) ? 1 : 0;
        ntot += 1;
        __syncwarp();
        if (MODE == 1 && (peers & lt) == 0) tab[warp][d] &= 0xffffu;  // clear masks (first peer)
        __syncwarp();
    }
    atomicAdd(bad, nbad);
    atomicAdd(total, ntot);
}

int main()
{
    unsigned long long *bad, *tot, hb, ht;
    cudaMalloc(&bad, 8);
    cudaMalloc(&tot, 8);
    for (int mode = 0; mode < 3; mode++)
        for (uint32_t nv : {1u, 2u, 4u, 16u, 64u, 256u}) {
            cudaMemset(bad, 0, 8);
            cudaMemset(tot, 0, 8);
            if (mode == 0) k_order<0><<<148 * 4, 512>>>(2000, nv, bad, tot);
            if (mode == 1) k_order<1><<<148 * 4, 512>>>(2000, nv, bad, tot);
            if (mode == 2) k_order<2><<<148 * 4, 512>>>(2000, nv, bad, tot);
            cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&ht, tot, 8, cudaMemcpyDeviceToHost);
            printf("mode %d values %3u: %llu of %llu lane-atomics NOT in lane order (%s)\n", mode, nv, hb, ht,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
