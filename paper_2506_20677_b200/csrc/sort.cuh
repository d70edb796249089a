// sort.cuh — K4 count_fill, K5 radix_hist, K6 onesweep pass.
//
// COUNTING  PAPER.md §III.F Listing 2 (lines 187-214): the histogram of
//           key - min (already built by ahs_features when shift = 0) and its
//           prefix give every key's final slot.  Keys only: K4 fills runs
//           out[o_v .. o_v + c_v) = min + v.  Key-value: one stable scatter
//           pass of K6 with the digit = key - min and bucket bases o_v.
// RADIX     §III.G (lines 218-251), base 256, d = ceil(log_256 k) digits
//           (Eq. 4) of u = key - min (R9).
// GENERAL   the QuickSort branch (§III.G.1) served by the same LSD radix on
//           the full 32-bit ordered key (4 passes).  LSD with stable passes
//           yields the unique stable sorted order, identical to the oracle.
//
// K6 is a onesweep digit pass (one read + one write of the keys per pass):
// each CTA takes the next tile from an atomic ticket, ranks its keys with
// warp-private digit counters + match.any (stable: warp-striped order), publishes
// per-digit tile counts, resolves its exclusive prefix by decoupled look-back
// over predecessor tiles, reorders the tile in shared memory and writes runs
// of equal digits to consecutive global addresses.
#pragma once

#include "common.cuh"

namespace ahs {

// ----------------------------------------------------------- status words
// status[tile][digit] = flag << 30 | count (count < 2^30 = AHS_MAX_N + 1)
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1u;

constexpr int kSortBlock = 512;
constexpr int kItemsKeys = 16;   // tile 8192 keys
constexpr int kItemsPairs = 8;   // tile 4096 pairs
constexpr int kMinTile = kSortBlock * kItemsPairs;

template <bool KV, int BITS>
struct OnesweepCfg {
    static constexpr int kBlock = kSortBlock;
    static constexpr int kWarps = kBlock / 32;
    static constexpr int kItems = KV ? kItemsPairs : kItemsKeys;
    static constexpr int kTile = kBlock * kItems;
    static constexpr int kBins = 1 << BITS;
    static constexpr uint32_t kMask = (uint32_t)kBins - 1u;
    // dynamic smem: stage keys | stage vals | whist[warps][bins] | 3 x bins
    static constexpr size_t kSmem = (size_t)kTile * 4 * (KV ? 2 : 1) + (size_t)kWarps * kBins * 4 +
                                    (size_t)3 * kBins * 4;
};

// ------------------------------------------------------------------ K5 ----
// One read of the keys: the `passes` digit histograms of v = (u ^ flip) - sub,
// smem-privatised (8 copies), flushed with global atomics into dhist (zeroed by
// the host's memset); the last CTA (atomic ticket) turns them into exclusive
// bucket bases, one warp per digit position.
constexpr int kRHBlock = 512;
constexpr int kRHUnroll = 4;
constexpr int kRHCopies = 8;

struct RadixHistOp {
    uint32_t *sh;  // [kRHCopies][4][256], this warp's copy
    uint32_t sub;
    int passes;
    __device__ __forceinline__ void operator()(uint32_t u, bool act)
    {
        if (!act) return;
        const uint32_t v = u - sub;
#pragma unroll
        for (int p = 0; p < 4; p++)
            if (p < passes) atomicAdd(&sh[p * 256 + ((v >> (8 * p)) & 255u)], 1u);
    }
};

template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK)
    k_radix_hist(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip, uint32_t sub,
                 int passes, uint32_t *__restrict__ dhist, uint32_t *__restrict__ bucket_base,
                 uint32_t *__restrict__ ticket)
{
    __shared__ uint32_t sh[kRHCopies * 4 * 256];
    __shared__ bool s_last;
    for (int i = threadIdx.x; i < kRHCopies * 4 * 256; i += BLOCK) sh[i] = 0u;
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    RadixHistOp op{sh + (warp % kRHCopies) * 1024, sub, passes};
    for_each_key<UNROLL>(keys, n, flip, op);
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += BLOCK) {
        uint32_t s = 0;
#pragma unroll
        for (int c = 0; c < kRHCopies; c++) s += sh[c * 1024 + i];
        if (s) atomicAdd(&dhist[i], s);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if ((int)warp < passes) {
        // exclusive scan of dhist[warp][0..256): lane owns 8 consecutive digits
        uint32_t c[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            c[j] = __ldcg(&dhist[warp * 256 + lane * 8 + j]);
            sum += c[j];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            bucket_base[warp * 256 + lane * 8 + j] = run;
            run += c[j];
        }
    }
}

// ------------------------------------------------------------------ K6 ----
// One stable digit pass.  Input transform on load: v = (key ^ in_flip) - in_sub;
// output transform on store: key = (v + out_add) ^ out_flip.  digit =
// (v >> shift) & (2^BITS - 1).  bucket_base[d] = first global slot of digit d.
template <bool KV, int BITS>
__global__ void __launch_bounds__(kSortBlock, 2)
    k_onesweep(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
               uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint32_t n,
               uint32_t shift, uint32_t in_flip, uint32_t in_sub, uint32_t out_flip,
               uint32_t out_add, const uint32_t *__restrict__ bucket_base,
               uint32_t *__restrict__ status, uint32_t *__restrict__ tile_ticket)
{
    using Cfg = OnesweepCfg<KV, BITS>;
    constexpr int TILE = Cfg::kTile, ITEMS = Cfg::kItems, BINS = Cfg::kBins, WARPS = Cfg::kWarps;
    constexpr uint32_t MASK = Cfg::kMask;
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *s_keys = smem;                                       // [TILE]
    uint32_t *s_vals = smem + TILE;                                // [TILE] (KV)
    uint32_t *s_whist = smem + TILE * (KV ? 2 : 1);                // [WARPS][BINS]
    uint32_t *s_count = s_whist + WARPS * BINS;                    // [BINS]
    uint32_t *s_start = s_count + BINS;                            // [BINS]
    uint32_t *s_gofs = s_start + BINS;                             // [BINS]
    __shared__ uint32_t s_tile;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_ticket, 1u);
    for (int i = tid; i < WARPS * BINS; i += kSortBlock) s_whist[i] = 0u;
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= gridDim.x) __trap();  // ticket not zeroed: refuse instead of waiting forever
    const uint32_t tile_base = tile * (uint32_t)TILE;
    const uint32_t tile_n = min((uint32_t)TILE, n - tile_base);

    // ---- load (warp-striped: item it of lane l is tile index w*32*ITEMS + it*32 + l)
    uint32_t v[ITEMS];
    uint32_t vv[KV ? ITEMS : 1];
    const uint32_t wbase = warp * 32u * ITEMS;
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        const uint32_t idx = wbase + it * 32u + lane;
        if (idx < tile_n) {
            v[it] = (ld_nc(keys_in + tile_base + idx) ^ in_flip) - in_sub;
            if constexpr (KV) vv[it] = ld_nc(vals_in + tile_base + idx);
        } else {
            v[it] = 0u;
            if constexpr (KV) vv[it] = 0u;
        }
    }

    // ---- rank within the warp (stable: items in order, lanes in order)
    uint32_t rank[ITEMS];
    uint32_t *wh = s_whist + warp * BINS;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        const uint32_t idx = wbase + it * 32u + lane;
        const bool valid = idx < tile_n;
        const uint32_t d = valid ? ((v[it] >> shift) & MASK) : (uint32_t)BINS;
        const uint32_t peers = __match_any_sync(kFull, d);
        const uint32_t leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader && valid) {
            base = wh[d];
            wh[d] = base + __popc(peers);
        }
        base = __shfl_sync(kFull, base, leader);
        rank[it] = base + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // ---- per digit: warp-exclusive offsets, tile count, publish aggregate
    for (int d = tid; d < BINS; d += kSortBlock) {
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < WARPS; w++) {
            const uint32_t t = s_whist[w * BINS + d];
            s_whist[w * BINS + d] = sum;
            sum += t;
        }
        s_count[d] = sum;
        st_relaxed(&status[(size_t)tile * BINS + d], (tile == 0 ? kFlagIncl : kFlagAgg) | sum);
    }
    __syncthreads();

    // ---- decoupled look-back (one thread per digit) + tile-local digit scan
    for (int d = tid; d < BINS; d += kSortBlock) {
        uint32_t excl = 0;
        if (tile > 0) {
            int j = (int)tile - 1;
            uint32_t spins = 0;
            while (true) {
                const uint32_t s = ld_relaxed(&status[(size_t)j * BINS + d]);
                const uint32_t flag = s & ~kCountMask;
                if (flag == 0u) {  // predecessor not published yet
                    // a predecessor always publishes (it took its ticket earlier and
                    // never waits before publishing); never hang the GPU on a bug
                    if (++spins > (1u << 28)) __trap();
                    continue;
                }
                excl += s & kCountMask;
                if (flag == kFlagIncl) break;
                j--;
            }
            st_relaxed(&status[(size_t)tile * BINS + d], kFlagIncl | (excl + s_count[d]));
        }
        s_gofs[d] = __ldg(&bucket_base[d]) + excl;
    }
    // local exclusive scan of s_count over digits (warp 0 .. ; BINS/32 per lane)
    if (warp == 0) {
        constexpr int PER = BINS / 32;
        uint32_t c[PER], sum = 0;
#pragma unroll
        for (int j = 0; j < PER; j++) {
            c[j] = s_count[lane * PER + j];
            sum += c[j];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int j = 0; j < PER; j++) {
            s_start[lane * PER + j] = run;
            run += c[j];
        }
    }
    __syncthreads();
    for (int d = tid; d < BINS; d += kSortBlock) s_gofs[d] -= s_start[d];

    // ---- scatter into shared memory in digit order
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        const uint32_t idx = wbase + it * 32u + lane;
        if (idx < tile_n) {
            const uint32_t d = (v[it] >> shift) & MASK;
            const uint32_t pos = s_start[d] + wh[d] + rank[it];
            s_keys[pos] = v[it];
            if constexpr (KV) s_vals[pos] = vv[it];
        }
    }
    __syncthreads();

    // ---- write out: consecutive tile slots of one digit -> consecutive global slots
    for (uint32_t i = tid; i < tile_n; i += kSortBlock) {
        const uint32_t x = s_keys[i];
        const uint32_t d = (x >> shift) & MASK;
        const uint32_t o = s_gofs[d] + i;
        keys_out[o] = (x + out_add) ^ out_flip;
        if constexpr (KV) vals_out[o] = s_vals[i];
    }
}

// ------------------------------------------------------------------ K4 ----
// Keys-only COUNTING: out[i] = min + v for scan[v] <= i < scan[v+1]
// (scan = exclusive prefix of the exact histogram, scan[nb] = n).  Each CTA
// owns a contiguous output chunk; thread 0 locates the chunk's first and last
// bins, every thread binary-searches within that (usually tiny) bin range and
// walks forward for its 4 consecutive outputs.  128-bit streaming stores.
constexpr int kFillBlock = 256;
constexpr int kFillVecPerThread = 8;
constexpr uint32_t kFillChunk = kFillBlock * kFillVecPerThread * 4;

__device__ __forceinline__ uint32_t upper_bin(const uint32_t *__restrict__ scan, uint32_t lo,
                                              uint32_t hi, uint32_t pos)
{
    // largest b in [lo, hi] with scan[b] <= pos (scan non-decreasing)
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1u) >> 1;
        if (__ldg(&scan[mid]) <= pos) lo = mid;
        else hi = mid - 1u;
    }
    return lo;
}

__global__ void __launch_bounds__(kFillBlock)
    k_count_fill(uint32_t *__restrict__ out, uint32_t n, const uint32_t *__restrict__ scan,
                 uint32_t nb, uint32_t out_flip, uint32_t out_add)
{
    __shared__ uint32_t s_lo, s_hi;
    // output positions are counted from the first 16-byte aligned element
    const uint32_t head = min(n, (uint32_t)(((16u - ((uintptr_t)out & 15u)) & 15u) >> 2));
    const uint32_t nvec = (n - head) >> 2;
    const uint32_t tail0 = head + 4u * nvec;
    const uint32_t c0 = blockIdx.x * kFillChunk;  // chunk in vector-body coordinates
    if (threadIdx.x == 0) {
        const uint32_t p0 = head + min(c0, 4u * nvec);
        const uint32_t p1 = head + min(c0 + kFillChunk, 4u * nvec);
        s_lo = upper_bin(scan, 0, nb - 1u, p0);
        s_hi = p1 > p0 ? upper_bin(scan, s_lo, nb - 1u, p1 - 1u) : s_lo;
    }
    __syncthreads();
    const uint32_t lo = s_lo, hi = s_hi;
    uint4 *vp = reinterpret_cast<uint4 *>(out + head);
#pragma unroll 2
    for (int j = 0; j < kFillVecPerThread; j++) {
        const uint32_t vi = (c0 >> 2) + j * kFillBlock + threadIdx.x;
        if (vi >= nvec) break;
        uint32_t pos = head + 4u * vi;
        uint32_t b = upper_bin(scan, lo, hi, pos);
        uint32_t r[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            while (__ldg(&scan[b + 1u]) <= pos + e) b++;
            r[e] = (b + out_add) ^ out_flip;
        }
        st_cs_v4(vp + vi, make_uint4(r[0], r[1], r[2], r[3]));
    }
    // unaligned head / tail (< 4 each)
    if (blockIdx.x == 0 && threadIdx.x < 8) {
        const uint32_t i = threadIdx.x < 4 ? threadIdx.x : tail0 + (threadIdx.x - 4);
        const bool act = threadIdx.x < 4 ? i < head : i < n;
        if (act) out[i] = (upper_bin(scan, 0, nb - 1u, i) + out_add) ^ out_flip;
    }
}

}  // namespace ahs
