// rankbench.cu — throughput of stable warp-level ranking of 8-bit digits on
// sm_100a (keys/clk/SM), the inner loop of the onesweep pass.  Each variant
// computes, per item, the peer mask (lanes with the same digit), the rank
// below me, and updates a warp-private digit counter in shared memory.
//   0 match.any   1 ballot x8 (compiler)   2 nibble lookup (8 ballots, lanes
//   build 16 hi + 16 lo masks, 2 shuffles)   3 smem atomicOr masks
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rb tools/rankbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr uint32_t FULL = 0xffffffffu;
constexpr int BLOCK = 512, WARPS = 16, ITEMS = 16;

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int V>
__global__ void __launch_bounds__(BLOCK, 2) k_rank(int reps, uint32_t *out)
{
    __shared__ uint32_t wh[WARPS][256];
    __shared__ uint32_t wm[WARPS][256];
    __shared__ uint2 wc[WARPS][256];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lt = lanemask_lt();
    for (int i = threadIdx.x; i < WARPS * 256; i += BLOCK) {
        (&wh[0][0])[i] = 0;
        (&wm[0][0])[i] = 0;
        (&wc[0][0])[i] = make_uint2(0, 0);
    }
    // variant 5: even warps rank with nibble ballots, odd warps with combined atomicOr
    const int mode = V == 5 ? ((warp & 1) ? 4 : 2) : (V == 6 ? ((warp % 4 == 0) ? 2 : 4) : V);
    __syncthreads();
    uint32_t key[ITEMS];
    uint32_t seed = hash32(blockIdx.x * BLOCK + threadIdx.x);
    for (int it = 0; it < ITEMS; it++) key[it] = hash32(seed + it);
    // nibble-lookup constants: lane builds the mask of nibble value (lane & 15)
    uint32_t m[4];
    for (int j = 0; j < 4; j++) m[j] = ((lane >> j) & 1) ? 0u : FULL;
    uint32_t acc = 0;
    for (int r = 0; r < reps; r++) {
#pragma unroll
        for (int it = 0; it < ITEMS; it++) {
            const uint32_t d = (key[it] >> ((r & 3) * 8)) & 255u;
            uint32_t peers;
            if (mode == 4) {
                atomicOr(&wc[warp][d].x, 1u << lane);
                __syncwarp();
                const uint2 e = wc[warp][d];
                __syncwarp();
                if (lane == 31 - __clz(e.x)) wc[warp][d] = make_uint2(0u, e.y + __popc(e.x));
                acc += e.y + __popc(e.x & lt);
                continue;
            }
            if (mode == 0) {
                peers = __match_any_sync(FULL, d);
            } else if (mode == 1) {
                peers = FULL;
#pragma unroll
                for (int b = 0; b < 8; b++) {
                    const uint32_t bb = __ballot_sync(FULL, (d >> b) & 1);
                    peers &= ((d >> b) & 1) ? bb : ~bb;
                }
            } else if (mode == 2) {
                uint32_t bl[8];
#pragma unroll
                for (int b = 0; b < 8; b++) bl[b] = __ballot_sync(FULL, (d >> b) & 1);
                const uint32_t mh = (bl[4] ^ m[0]) & (bl[5] ^ m[1]) & (bl[6] ^ m[2]) & (bl[7] ^ m[3]);
                const uint32_t ml = (bl[0] ^ m[0]) & (bl[1] ^ m[1]) & (bl[2] ^ m[2]) & (bl[3] ^ m[3]);
                peers = __shfl_sync(FULL, mh, d >> 4) & __shfl_sync(FULL, ml, d & 15);
            } else {
                atomicOr(&wm[warp][d], 1u << lane);
                __syncwarp();
                peers = wm[warp][d];
                __syncwarp();
            }
            const uint32_t leader = 31 - __clz(peers);
            uint32_t base = 0;
            if (lane == leader) {
                base = wh[warp][d];
                wh[warp][d] = base + __popc(peers);
                if (mode == 3) wm[warp][d] = 0;
            }
            base = __shfl_sync(FULL, base, leader);
            acc += base + __popc(peers & lt);
            __syncwarp();
        }
    }
    out[blockIdx.x * BLOCK + threadIdx.x] = acc;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out;
    cudaMalloc(&out, sms * 8 * BLOCK * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 256;
    for (int v = 0; v < 7; v++) {
        auto run = [&] {
            int g = sms * 2;
            if (v == 0) k_rank<0><<<g, BLOCK>>>(reps, out);
            if (v == 1) k_rank<1><<<g, BLOCK>>>(reps, out);
            if (v == 2) k_rank<2><<<g, BLOCK>>>(reps, out);
            if (v == 3) k_rank<3><<<g, BLOCK>>>(reps, out);
            if (v == 4) k_rank<4><<<g, BLOCK>>>(reps, out);
            if (v == 5) k_rank<5><<<g, BLOCK>>>(reps, out);
            if (v == 6) k_rank<6><<<g, BLOCK>>>(reps, out);
        };
        run();
        cudaEventRecord(a);
        run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double keys = (double)sms * 2 * BLOCK * ITEMS * reps;
        static uint32_t h[148 * 2 * BLOCK];
        cudaMemcpy(h, out, sms * 2 * BLOCK * 4, cudaMemcpyDeviceToHost);
        unsigned long long cs = 0;
        for (int i = 0; i < sms * 2 * BLOCK; i++) cs += h[i];
        printf("variant %d: %.1f Gkeys/s ranked = %.2f keys/clk/SM @1.9GHz checksum %llu (err %s)\n", v,
               keys / ms / 1e6, keys / ms / 1e6 / sms / 1.9, cs, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
