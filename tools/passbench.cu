// passbench.cu — development tool: one onesweep digit pass (K6) in isolation,
// several launch configurations, checked against a host counting sort, plus
// CUB's DeviceRadixSort on the same data as an outside reference point.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o tools/pb tools/passbench.cu
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "onesweep_p.cuh"
#include "onesweep_b.cuh"
#include "../paper_2506_20677_b200/csrc/onesweep2.cuh"

using namespace ahs;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__host__ __device__ inline uint32_t hash32(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// dist 0: uniform 32-bit; 1: 64 distinct values Zipf-ish (low-entropy digit); 2: constant digit
__global__ void k_gen(uint32_t *k, uint32_t *v, uint32_t n, int dist, uint32_t seed)
{
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t x = hash32(i * 2654435761u + seed);
        if (dist == 1) {
            uint32_t u = hash32(x) & 0xffffu;
            uint32_t r = 0;
            while (r < 63 && u < (65536u >> (r / 4 + 1))) r++;  // skewed
            x = (r << 2) | (x & 0xffffff00u);
        } else if (dist == 2) {
            x = (x & 0xffffff00u) | 42u;
        } else if (dist == 3) {  // ascending (presorted) keys
            x = i;
        }
        k[i] = x;
        v[i] = i;
    }
}

__global__ void k_dhist(const uint32_t *k, uint32_t n, uint32_t shift, uint32_t *hist)
{
    __shared__ uint32_t sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&sh[(k[i] >> shift) & 255u], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) atomicAdd(&hist[i], sh[i]);
}

__global__ void k_flush(uint32_t *p, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

struct Bufs {
    uint32_t *k, *v, *ko, *vo, *bb, *status, *ticket, *flush;
    size_t flush_n;
};

static int g_only = -1, g_idx = 0;
static bool g_noflush = false;  // env PB_NOFLUSH=1: the pass input stays L2-warm (as inside a sort)
static bool g_mid = false;      // env PB_MID=1: run as a middle pass of a chain (no key transforms)

template <bool KV>
float run_kern(const Bufs &B, uint32_t n, uint32_t shift, int sms, int reps, bool check,
               const std::vector<uint32_t> &hk, const std::vector<uint32_t> &hbase, const void *kern, size_t smem,
               int tile, int block, const char *name, uint32_t bins = 256)
{
    if (g_only >= 0 && g_idx++ != g_only) return 0.f;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem));
    const uint32_t tiles = (n + tile - 1) / tile;
    if (getenv("PB_OCC")) occ = std::min(occ, atoi(getenv("PB_OCC")));  // fewer CTAs per SM
    const uint32_t grid = std::min<uint32_t>(tiles, (uint32_t)(occ * sms));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ts;
    for (int r = 0; r < reps + 2; r++) {
        if (!g_noflush) k_flush<<<sms * 4, 512>>>(B.flush, B.flush_n);
        CK(cudaMemsetAsync(B.status, 0, (size_t)tiles * bins * 4));
        CK(cudaMemsetAsync(B.ticket, 0, 4));
        CK(cudaEventRecord(a));
        PassArgs pa{};
        pa.keys_in = B.k;
        pa.vals_in = B.v;
        pa.keys_out = B.ko;
        pa.vals_out = B.vo;
        pa.keys_tmp = B.ko;
        pa.vals_tmp = B.vo;
        pa.n = n;
        pa.pass = 0;
        pa.npasses = 1;
        if (g_mid) {  // executed pass 1 of 3: reads keys_out, writes keys_tmp, no transforms
            pa.pass = 1;
            pa.npasses = 3;
            pa.keys_out = B.k;
            pa.vals_out = B.v;
        }
        pa.shift = shift;
        pa.bucket_base = B.bb;
        pa.status = B.status;
        pa.ticket = B.ticket;
        pa.plan = nullptr;
        { void *args[] = {&pa}; CK(cudaLaunchKernel(kern, dim3(grid), dim3(block), args, smem, 0)); }
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r >= 2) ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const float med = ts[ts.size() / 2];
#ifdef AHS_PHASE_STATS
    {
        unsigned long long ph[8];
        CK(cudaMemcpyFromSymbol(ph, g_phase_cycles, sizeof(ph)));
        const double per = (double)tiles * (reps + 2);
        const char *nm[7] = {"tma wait", "early counts", "totals+scan", "offsets", "rank+scatter",
                             "look-back+sync", "write-out+sync"};
        double tot = 0;
        for (int k = 0; k < 7; k++) tot += ph[k] / per;
        printf("  phases (cycles per tile, thread 0):");
        for (int k = 0; k < 7; k++) printf(" %s %.0f (%.0f%%)", nm[k], ph[k] / per, 100.0 * ph[k] / per / tot);
        printf("  total %.0f\n", tot);
        memset(ph, 0, sizeof(ph));
        CK(cudaMemcpyToSymbol(g_phase_cycles, ph, sizeof(ph)));
        unsigned long long lp[4];
        CK(cudaMemcpyFromSymbol(lp, g_lb_probe, sizeof(lp)));
        printf("  look-back (thread 0): %.2f rounds, %.0f cycles, %.0f cycles/round, %.2f empty rounds per tile\n",
               (double)lp[1] / lp[0], (double)lp[2] / lp[0], (double)lp[2] / lp[1], (double)lp[3] / lp[0]);
        memset(lp, 0, sizeof(lp));
        CK(cudaMemcpyToSymbol(g_lb_probe, lp, sizeof(lp)));
    }
#endif
#ifdef AHS_LB_STATS
    {
        unsigned long long st[4];
        CK(cudaMemcpyFromSymbol(st, g_lb_stats, sizeof(st)));
        printf("  look-back (W=%d): per digit-tile %.2f rounds, %.2f empty rounds, %.1f statuses\n", kLookback,
               (double)st[1] / st[0], (double)st[2] / st[0], (double)st[3] / st[0]);
        memset(st, 0, sizeof(st));
        CK(cudaMemcpyToSymbol(g_lb_stats, st, sizeof(st)));
    }
#endif
    bool ok = true;
    if (check) {
        std::vector<uint32_t> got(n), gotv(n), pos(hbase);
        CK(cudaMemcpy(got.data(), B.ko, n * 4ull, cudaMemcpyDeviceToHost));
        if (KV) CK(cudaMemcpy(gotv.data(), B.vo, n * 4ull, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < n && ok; i++) {
            const uint32_t p = pos[(hk[i] >> shift) & (bins - 1)]++;
            if (got[p] != hk[i] || (KV && gotv[p] != i)) {
                printf("  MISMATCH at out %u (in %u): got %08x want %08x\n", p, i, got[p], hk[i]);
                ok = false;
            }
        }
    }
    const double bytes = (KV ? 16.0 : 8.0) * n;
    printf("  %-32s tile %5d occ %d grid %4u: %8.1f us  %7.1f GB/s  %6.1f Gkeys/s  "
           "%.2f keys/clk/SM@1.9 max %.1f us %s\n",
           name, tile, occ, grid, med * 1e3, bytes / med / 1e6,
           n / med / 1e6, n / med / 1e6 / sms / 1.9, ts.back() * 1e3, check ? (ok ? "ok" : "FAIL") : "");
    return med;
}

template <bool KV, int BLOCK, int ITEMS, int MINB, int RANK = kRankMasked>
float run_cfg(const Bufs &B, uint32_t n, uint32_t shift, int sms, int reps, bool check,
              const std::vector<uint32_t> &hk, const std::vector<uint32_t> &hbase)
{
    using C = Onesweep<KV, BLOCK, ITEMS, RANK>;
    char nm[96];
    snprintf(nm, sizeof nm, "%s<%s,B%d,I%d,minb%d>", RANK == kRankOrdered ? "ordered" : "masked", KV ? "kv" : "k",
             BLOCK, ITEMS, MINB);
    return run_kern<KV>(B, n, shift, sms, reps, check, hk, hbase,
                        (const void *)k_onesweep<KV, BLOCK, ITEMS, MINB, RANK>, C::kSmem, C::kTile, BLOCK, nm);
}

template <bool KV, int NW, int ITEMS, int LBW, int W = 8>
float run_p(const Bufs &B, uint32_t n, uint32_t shift, int sms, int reps, bool check,
            const std::vector<uint32_t> &hk, const std::vector<uint32_t> &hbase)
{
    using C = OnesweepP<KV, NW, ITEMS, LBW>;
    char nm[96];
    snprintf(nm, sizeof nm, "P<%s,NW%d,I%d,LB%d,W%d>", KV ? "kv" : "k", NW, ITEMS, LBW, W);
    return run_kern<KV>(B, n, shift, sms, reps, check, hk, hbase,
                        (const void *)k_onesweep_p<KV, NW, ITEMS, LBW, W>, C::kSmem, C::kTile, C::kBlock, nm);
}

template <bool KV, int BLOCK, int ITEMS, int MINB>
float run_b(const Bufs &B, uint32_t n, uint32_t shift, int sms, int reps, bool check,
            const std::vector<uint32_t> &hk, const std::vector<uint32_t> &hbase)
{
    using C = OnesweepB<KV, BLOCK, ITEMS>;
    char nm[96];
    snprintf(nm, sizeof nm, "bulk<%s,B%d,I%d,minb%d>", KV ? "kv" : "k", BLOCK, ITEMS, MINB);
    return run_kern<KV>(B, n, shift, sms, reps, check, hk, hbase,
                        (const void *)k_onesweep_b<KV, BLOCK, ITEMS, MINB>, C::kSmem, C::kTile, BLOCK, nm);
}

template <bool KV, int BLOCK, int ITEMS, int BITS = 8, int HOT = kHotDefault>
float run2(const Bufs &B, uint32_t n, uint32_t shift, int sms, int reps, bool check,
           const std::vector<uint32_t> &hk, const std::vector<uint32_t> &hbase)
{
    using C = Onesweep2<KV, BLOCK, ITEMS, BITS, uint32_t, uint32_t, HOT>;
    char nm[96];
    snprintf(nm, sizeof nm, "v2<%s,B%d,I%d,b%d,hot%x>", KV ? "kv" : "k", BLOCK, ITEMS, BITS, HOT);
    return run_kern<KV>(B, n, shift, sms, reps, check, hk, hbase,
                        (const void *)k_onesweep2<KV, BLOCK, ITEMS, (BLOCK == 256 && BITS == 8 ? 4 : 2), BITS,
                                                  uint32_t, uint32_t, HOT>,
                        C::kSmem, C::kTile, BLOCK, nm, 1u << BITS);
}

template <bool KV>
void run_cub(const Bufs &B, uint32_t n, int begin_bit, int end_bit, int sms, int reps)
{
    size_t tb = 0;
    if (KV)
        cub::DeviceRadixSort::SortPairs(nullptr, tb, B.k, B.ko, B.v, B.vo, (int)n, begin_bit, end_bit);
    else
        cub::DeviceRadixSort::SortKeys(nullptr, tb, B.k, B.ko, (int)n, begin_bit, end_bit);
    void *tmp;
    CK(cudaMalloc(&tmp, tb));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ts;
    for (int r = 0; r < reps + 2; r++) {
        k_flush<<<sms * 4, 512>>>(B.flush, B.flush_n);
        CK(cudaEventRecord(a));
        if (KV)
            cub::DeviceRadixSort::SortPairs(tmp, tb, B.k, B.ko, B.v, B.vo, (int)n, begin_bit, end_bit);
        else
            cub::DeviceRadixSort::SortKeys(tmp, tb, B.k, B.ko, (int)n, begin_bit, end_bit);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r >= 2) ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const float med = ts[ts.size() / 2];
    const int passes = (end_bit - begin_bit + 7) / 8;
    const double bytes = (KV ? 4.0 + 16.0 * passes : 4.0 + 8.0 * passes) * n;
    printf("  CUB %s bits [%d,%d): %8.1f us  %6.1f Gkeys/s  (%.0f GB/s at (%s) bytes)\n", KV ? "pairs" : "keys",
           begin_bit, end_bit, med * 1e3, n / med / 1e6, bytes / med / 1e6, KV ? "4+16p" : "4+8p");
    CK(cudaFree(tmp));
}

int main(int argc, char **argv)
{
    const uint32_t n = argc > 1 ? (uint32_t)atol(argv[1]) : (1u << 26);
    const int dist = argc > 2 ? atoi(argv[2]) : 0;
    const int reps = argc > 3 ? atoi(argv[3]) : 10;
    const bool cub = argc > 4 ? atoi(argv[4]) != 0 : true;
    g_only = argc > 5 ? atoi(argv[5]) : -1;
    g_noflush = getenv("PB_NOFLUSH") && getenv("PB_NOFLUSH")[0] == '1';
    g_mid = getenv("PB_MID") && getenv("PB_MID")[0] == '1';
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    Bufs B;
    CK(cudaMalloc(&B.k, n * 4ull));
    CK(cudaMalloc(&B.v, n * 4ull));
    CK(cudaMalloc(&B.ko, n * 4ull));
    CK(cudaMalloc(&B.vo, n * 4ull));
    CK(cudaMalloc(&B.bb, 2048 * 4));
    CK(cudaMalloc(&B.status, ((size_t)n / 1024 + 16) * 2048 * 4));
    CK(cudaMalloc(&B.ticket, 64));
    B.flush_n = 64u << 20;  // 256 MiB
    CK(cudaMalloc(&B.flush, B.flush_n * 4));
    k_gen<<<sms * 8, 256>>>(B.k, B.v, n, dist, 12345u);
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> hk(n);
    CK(cudaMemcpy(hk.data(), B.k, n * 4ull, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> shifts = {0u, 8u};
    if (dist == 4) {  // cfg3-like: j * 2^18, j ~ Zipf(1.1) on [0, 4096) by inverse CDF (digits 2 and 3 vary)
        std::vector<double> cdf(4096);
        double acc = 0.0;
        for (int j = 0; j < 4096; j++) cdf[j] = (acc += std::pow(j + 1.0, -1.1));
        for (int j = 0; j < 4096; j++) cdf[j] /= acc;
        cdf[4095] = 1.0;
        for (uint32_t i = 0; i < n; i++) {
            const double u = (hash32(i * 2654435761u + 777u) >> 8) * (1.0 / 16777216.0);
            const uint32_t j = (uint32_t)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
            hk[i] = std::min(j, 4095u) << 18;
        }
        CK(cudaMemcpy(B.k, hk.data(), n * 4ull, cudaMemcpyHostToDevice));
        shifts = {16u, 24u};
    }
    printf("n = %u, dist %d, %d SMs\n", n, dist, sms);
    if (getenv("PB_SHIFTS")) {  // e.g. PB_SHIFTS=24 or 16,24
        shifts.clear();
        for (const char *q = getenv("PB_SHIFTS"); *q;) {
            shifts.push_back((uint32_t)strtoul(q, (char **)&q, 10));
            if (*q == ',') q++;
        }
    }
    if (getenv("PB_SKIP8")) shifts.clear();
    for (uint32_t shift : shifts)
        if (g_only < 0 || shift == shifts[0]) {
        std::vector<uint32_t> hist(256, 0), base(256);
        for (uint32_t i = 0; i < n; i++) hist[(hk[i] >> shift) & 255u]++;
        uint32_t run = 0, mx = 0;
        for (int d = 0; d < 256; d++) {
            base[d] = run;
            run += hist[d];
            mx = std::max(mx, hist[d]);
        }
        CK(cudaMemcpy(B.bb, base.data(), 1024, cudaMemcpyHostToDevice));
        printf("digit shift %u (max digit share %.3f)\n", shift, (double)mx / n);
        g_idx = 0;
        run_cfg<false, 512, 18, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
        if (getenv("PB_BULK")) {  // K6b: TMA bulk-store write-out per digit run
            run_b<false, 512, 18, 2>(B, n, shift, sms, reps, true, hk, base);
            run_b<false, 512, 16, 2>(B, n, shift, sms, reps, true, hk, base);
            run_b<false, 384, 16, 3>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<true, 384, 16, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_b<true, 384, 12, 2>(B, n, shift, sms, reps, true, hk, base);
            run_b<true, 256, 20, 2>(B, n, shift, sms, reps, true, hk, base);
            run_b<true, 256, 18, 2>(B, n, shift, sms, reps, true, hk, base);
            continue;
        }
        if (getenv("PB_SHAPES")) {  // keys-only launch shapes: tile vs CTAs per SM
            run_cfg<false, 256, 18, 4, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 256, 24, 3, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 384, 16, 3, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 512, 24, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 512, 12, 3, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
        }
        run2<false, 512, 18, 8, 0>(B, n, shift, sms, reps, true, hk, base);
        run2<false, 512, 18, 8, hotcfg(1, 3, false)>(B, n, shift, sms, reps, true, hk, base);
        run2<false, 512, 18, 8, hotcfg(4, 3, false)>(B, n, shift, sms, reps, true, hk, base);
        run2<false, 512, 18, 8, hotcfg(2, 4, false)>(B, n, shift, sms, reps, true, hk, base);
        run_cfg<true, 384, 16, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
        if (getenv("PB_SHAPES3")) {  // keys-only: 256 threads, 2 CTAs per SM, large tiles
            run_cfg<false, 256, 32, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 256, 36, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 256, 40, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 256, 44, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<false, 384, 24, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
        }
        if (getenv("PB_SHAPES2")) {  // key-value launch shapes with packed slots (72 registers)
            run_cfg<true, 512, 11, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<true, 256, 24, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<true, 256, 25, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<true, 384, 15, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
        }
        if (getenv("PB_SHAPES")) {  // key-value launch shapes
            run_cfg<true, 256, 15, 3, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<true, 256, 20, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<true, 512, 12, 2, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
            run_cfg<true, 384, 10, 3, kRankOrdered>(B, n, shift, sms, reps, true, hk, base);
        }
        run2<true, 384, 16, 8, hotcfg(1, 3, false)>(B, n, shift, sms, reps, true, hk, base);
        run2<true, 384, 16, 8, hotcfg(4, 3, false)>(B, n, shift, sms, reps, true, hk, base);
    }
    // wider digits (low BITS bits): KV counting with k <= 1024 (10 bits), the 11-bit experiment
    if (getenv("PB_WIDE")) {
        for (int bits : {9, 10, 11}) {
            const uint32_t bins = 1u << bits;
            std::vector<uint32_t> hist(bins, 0), base(bins);
            for (uint32_t i = 0; i < n; i++) hist[hk[i] & (bins - 1)]++;
            uint32_t run = 0;
            for (uint32_t d = 0; d < bins; d++) {
                base[d] = run;
                run += hist[d];
            }
            CK(cudaMemcpy(B.bb, base.data(), bins * 4, cudaMemcpyHostToDevice));
            printf("digit bits %d, shift 0\n", bits);
            g_idx = 0;
            if (bits == 9) {
                run2<false, 256, 36, 9>(B, n, 0, sms, reps, true, hk, base);
                run2<false, 256, 32, 9>(B, n, 0, sms, reps, true, hk, base);
                run2<false, 256, 24, 9>(B, n, 0, sms, reps, true, hk, base);
                run2<false, 256, 18, 9>(B, n, 0, sms, reps, true, hk, base);
            } else if (bits == 10) {
                run2<false, 512, 16, 10>(B, n, 0, sms, reps, true, hk, base);
                run2<true, 512, 8, 10>(B, n, 0, sms, reps, true, hk, base);
                run2<true, 512, 10, 10>(B, n, 0, sms, reps, true, hk, base);
                run2<true, 256, 16, 10>(B, n, 0, sms, reps, true, hk, base);
            } else {
                run2<false, 512, 16, 11>(B, n, 0, sms, reps, true, hk, base);
                run2<false, 512, 12, 11>(B, n, 0, sms, reps, true, hk, base);
                run2<false, 512, 24, 11>(B, n, 0, sms, reps, true, hk, base);
            }
        }
    }
    if (cub) {
        run_cub<false>(B, n, 0, 32, sms, reps);
        run_cub<false>(B, n, 0, 8, sms, reps);
        run_cub<true>(B, n, 0, 32, sms, reps);
    }
    return 0;
}
