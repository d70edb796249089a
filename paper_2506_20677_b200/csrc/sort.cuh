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
#include "features.cuh"

namespace ahs {

// ----------------------------------------------------------- status words
// status[tile][digit] = flag << 30 | count (count < 2^30 = AHS_MAX_N + 1)
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1u;

constexpr int kSortBlock = 512;
constexpr int kSortWarps = kSortBlock / 32;
constexpr int kItemsKeys = 16;  // tile 8192 keys
constexpr int kItemsPairs = 8;  // tile 4096 pairs
constexpr int kMinTile = kSortBlock * kItemsPairs;
constexpr int kLookback = 8;    // predecessor statuses loaded per look-back round
constexpr int kBins = 256;      // 8-bit digits

template <bool KV>
struct OnesweepCfg {
    static constexpr int kItems = KV ? kItemsPairs : kItemsKeys;
    static constexpr int kTile = kSortBlock * kItems;
    // dynamic shared memory:
    //   s_k    [TILE]          tile keys (TMA / loads), reused for the reordered keys
    //   s_vin  [TILE]    (KV)  tile values
    //   s_vout [TILE]    (KV)  reordered values
    //   s_wc   [WARPS][256]    uint2 {peer mask, running count} per warp and digit
    //   s_off  [WARPS][256]    combined scatter offset per warp and digit
    //   s_count, s_start, s_gofs [256]
    static constexpr size_t kKeyBytes = (size_t)kTile * 4 * (KV ? 3 : 1);
    static constexpr size_t kSmem = kKeyBytes + (size_t)kSortWarps * kBins * 8 + (size_t)kSortWarps * kBins * 4 +
                                    (size_t)3 * kBins * 4;
};

// ------------------------------------------------------------------ K5 ----
// Digit histograms of v = (key ^ flip) - min for the `passes` 8-bit digits.
// Digits whose bits lie inside [fshift, 32) are read off the feature
// histogram (ws, exact counts of v >> fshift): a bucket's keys share those
// bits.  Only when fshift > 0 (k > 2^16) are the keys read again, for the
// joint histogram of their low 16 bits (digits 0 and 1) in 2^16 packed
// guard-bit counters: ONE shared atomic per key instead of one per digit
// (the kernel is shared-atomic bound otherwise), with the same run merging
// as feat_hist.  Marginals are flushed with global atomics into dhist (zeroed
// by the host's memset); the last CTA turns them into exclusive bucket bases.
constexpr int kRHBlock = 512;
constexpr int kRHChunk = 40 * 1024;  // 5 vectors per thread
constexpr int kRHStages = 2;
constexpr int kRHSmem = kHistBins + kRHStages * (kRHChunk + 16);

struct JointAdd {  // packed joint counter; overflow goes straight to the marginals
    uint32_t *sh, *dig0, *dig1;
    __device__ __forceinline__ void operator()(uint32_t b, uint32_t c) const
    {
        const uint32_t sft = (b & 1u) << 4;
        const uint32_t old = atomicAdd(&sh[b >> 1], c << sft);
        const uint32_t h = (old >> sft) & 0xffffu;
        if (h < 0x8000u && h + c >= 0x8000u) {
            atomicSub(&sh[b >> 1], 0x8000u << sft);
            atomicAdd(&dig0[b & 255u], 0x8000u);
            atomicAdd(&dig1[b >> 8], 0x8000u);
        }
    }
};

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1)
    k_radix_hist(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip, uint32_t sub, int passes,
                 const uint32_t *__restrict__ fhist, uint32_t nb, uint32_t fshift,
                 uint32_t *__restrict__ dhist, uint32_t *__restrict__ bucket_base,
                 uint32_t *__restrict__ ticket)
{
    extern __shared__ __align__(128) uint32_t sh[];
    __shared__ uint32_t s_dig[4][256];
    __shared__ __align__(8) uint64_t bars[kRHStages];
    __shared__ bool s_last;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const bool from_keys = fshift > 0u;  // digits 0 and 1 need the keys
    for (int i = threadIdx.x; i < 4 * 256; i += BLOCK) (&s_dig[0][0])[i] = 0u;
    if (from_keys)
        for (int i = threadIdx.x; i < (int)kHistWords; i += BLOCK) sh[i] = 0u;
    __syncthreads();

    if (from_keys) {
        const JointAdd add{sh, s_dig[0], s_dig[1]};
        const uint32_t c0 = sub - flip;
        const VecSplit sp = vec_split(keys, n);
        const uint4 *body = reinterpret_cast<const uint4 *>(keys + sp.head);
        uint8_t *stage = reinterpret_cast<uint8_t *>(sh) + kHistBins;
        stream_chunks<kRHStages, kRHChunk>(body, sp.nvec, stage, bars, [&](const uint4 *c, uint32_t nv, uint64_t) {
            for (uint32_t j0 = 0; j0 < nv; j0 += BLOCK) {
                const uint32_t j = j0 + threadIdx.x;
                const bool act = j < nv;
                const uint4 x = act ? c[j] : make_uint4(0u, 0u, 0u, 0u);
                // bins = low 16 bits of v = key - (sub - flip)  (mod 2^32)
                hist_vec(add,
                         make_uint4((x.x - c0) & 0xffffu, (x.y - c0) & 0xffffu, (x.z - c0) & 0xffffu,
                                    (x.w - c0) & 0xffffu),
                         act, 0u);
            }
        });
        if (blockIdx.x == 0 && warp == 0) {  // head / tail keys, one per lane
            const uint64_t i = lane < 3 ? lane : sp.tail0 + (lane - 3);
            const bool act = lane < 3 ? i < sp.head : (lane < 6 && i < n);
            if (act) add((keys[i] - c0) & 0xffffu, 1u);
        }
        __syncthreads();
        // marginals: threads 0..255 own digit-0 value t, 256..511 digit-1 value t - 256
        if (threadIdx.x < 512) {
            const uint32_t t = threadIdx.x & 255u;
            uint32_t sum = 0;
            if (threadIdx.x < 256) {
                for (uint32_t d1 = 0; d1 < 256; d1++) {
                    const uint32_t b = (d1 << 8) | t;
                    sum += (sh[b >> 1] >> ((b & 1u) << 4)) & 0xffffu;
                }
                atomicAdd(&s_dig[0][t], sum);
            } else {
                for (uint32_t w = t << 7; w < (t << 7) + 128u; w++) {
                    const uint32_t x = sh[w];
                    sum += (x & 0xffffu) + (x >> 16);
                }
                atomicAdd(&s_dig[1][t], sum);
            }
        }
    }
    // digits inside the feature buckets: this CTA's slice of the bins
    for (uint32_t b = blockIdx.x * BLOCK + threadIdx.x; b < nb; b += gridDim.x * BLOCK) {
        const uint32_t c = __ldg(&fhist[b]);
        if (!c) continue;
        const uint32_t base = b << fshift;
#pragma unroll
        for (int p = 0; p < 4; p++)
            if (p < passes && (uint32_t)(8 * p) >= fshift && !(from_keys && p < 2))
                atomicAdd(&s_dig[p][(base >> (8 * p)) & 255u], c);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += BLOCK) {
        const uint32_t v = (&s_dig[0][0])[i];
        if (v) atomicAdd(&dhist[i], v);
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
// One stable 8-bit digit pass.  Input transform on load: v = (key ^ in_flip) -
// in_sub; output transform on store: key = (v + out_add) ^ out_flip; digit =
// byte (shift / 8) of v.  bucket_base[d] = first global slot of digit d.
//
// Tile load: one TMA bulk copy (keys, and values for KV) when the input is
// 16-byte aligned and the tile full, else coalesced loads.  Ranking (stable,
// warp-striped order): per item, every lane sets its bit in the warp's
// {mask, count} word of its digit with a shared atomicOr, reads the word back
// (peers = lanes with the same digit, count = earlier items' total), and the
// highest peer lane writes {0, count + popc(peers)}.  On sm_100 this is ~2x
// the throughput of ballot-based ranking and ~4x match.any (tools/rankbench.cu).
__device__ __forceinline__ uint32_t digit8(uint32_t v, uint32_t shift)
{
    return __byte_perm(v, 0u, 0x4440u | (shift >> 3));
}

template <bool KV>
__global__ void __launch_bounds__(kSortBlock, 2)
    k_onesweep(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
               uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint32_t n,
               uint32_t shift, uint32_t in_flip, uint32_t in_sub, uint32_t out_flip,
               uint32_t out_add, const uint32_t *__restrict__ bucket_base,
               uint32_t *__restrict__ status, uint32_t *__restrict__ tile_ticket, uint32_t tma_ok)
{
    using Cfg = OnesweepCfg<KV>;
    constexpr int TILE = Cfg::kTile, ITEMS = Cfg::kItems, WARPS = kSortWarps;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint32_t *s_k = reinterpret_cast<uint32_t *>(smem_raw);
    uint32_t *s_vin = s_k + TILE;
    uint32_t *s_vout = s_vin + TILE;
    uint2 *s_wc = reinterpret_cast<uint2 *>(smem_raw + Cfg::kKeyBytes);
    uint32_t *s_off = reinterpret_cast<uint32_t *>(s_wc + WARPS * kBins);
    uint32_t *s_count = s_off + WARPS * kBins;
    uint32_t *s_start = s_count + kBins;
    uint32_t *s_gofs = s_start + kBins;
    __shared__ uint32_t s_tile;
    __shared__ __align__(8) uint64_t s_bar;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) {
        s_tile = atomicAdd(tile_ticket, 1u);
        mbar_init(&s_bar, 1);
        mbar_fence_init();
    }
    for (int i = tid; i < WARPS * kBins / 2; i += kSortBlock)
        reinterpret_cast<uint4 *>(s_wc)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= gridDim.x) __trap();  // ticket not zeroed: refuse instead of waiting forever
    const uint32_t tile_base = tile * (uint32_t)TILE;
    const uint32_t tile_n = min((uint32_t)TILE, n - tile_base);

    // ---- tile load
    if (tma_ok && tile_n == (uint32_t)TILE) {
        if (tid == 0) {
            mbar_expect_tx(&s_bar, (uint32_t)TILE * 4u * (KV ? 2u : 1u));
            tma_load_1d(s_k, keys_in + tile_base, (uint32_t)TILE * 4u, &s_bar);
            if constexpr (KV) tma_load_1d(s_vin, vals_in + tile_base, (uint32_t)TILE * 4u, &s_bar);
        }
        mbar_wait(&s_bar, 0);
    } else {
        for (uint32_t i = tid; i < tile_n; i += kSortBlock) {
            s_k[i] = ld_nc(keys_in + tile_base + i);
            if constexpr (KV) s_vin[i] = ld_nc(vals_in + tile_base + i);
        }
        __syncthreads();
    }

    // ---- rank within the warp (stable: items in order, lanes in order)
    uint32_t v[ITEMS], rank2[ITEMS / 2];  // ranks < TILE <= 2^13, packed two per register
    uint2 *wc = s_wc + warp * kBins;
    const uint32_t lt = lanemask_lt();
    const uint32_t wbase = warp * 32u * ITEMS;
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        const uint32_t idx = wbase + it * 32u + lane;
        const bool valid = idx < tile_n;
        v[it] = valid ? ((s_k[idx] ^ in_flip) - in_sub) : 0u;
        const uint32_t d = digit8(v[it], shift);
        uint32_t r;
        // one digit across the warp (constant digits, sorted runs): no atomics
        // (same-address shared atomics serialise)
        const uint32_t d0 = __shfl_sync(kFull, d, 0);
        if (__all_sync(kFull, !valid || d == d0)) {
            const uint32_t vm = __ballot_sync(kFull, valid);
            const uint32_t base = wc[d0].y;
            __syncwarp();
            if (lane == 0) wc[d0].y = base + __popc(vm);
            r = base + __popc(vm & lt);
        } else {
            if (valid) atomicOr(&wc[d].x, 1u << lane);
            __syncwarp();
            const uint2 e = valid ? wc[d] : make_uint2(0u, 0u);
            __syncwarp();
            if (valid && lane == 31u - __clz(e.x)) wc[d] = make_uint2(0u, e.y + __popc(e.x));
            r = e.y + __popc(e.x & lt);
        }
        if (it & 1) rank2[it / 2] |= r << 16;
        else rank2[it / 2] = r;
        __syncwarp();
    }
    __syncthreads();

    // ---- per digit: warp-exclusive offsets, tile count, publish aggregate
    if (tid < kBins) {
        const uint32_t d = tid;
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < WARPS; w++) {
            const uint32_t t = s_wc[w * kBins + d].y;
            s_off[w * kBins + d] = sum;
            sum += t;
        }
        s_count[d] = sum;
        st_relaxed(&status[(size_t)tile * kBins + d], (tile == 0 ? kFlagIncl : kFlagAgg) | sum);
    }
    __syncthreads();

    // ---- decoupled look-back (threads 0..255, one digit each) || local digit scan (warp 8).
    // Each round loads the statuses of kLookback predecessor tiles at once and
    // consumes them newest-first: AGG counts accumulate, the first INCL ends
    // the walk, an unpublished one is re-read next round.  Tile -1 is INCL 0.
    if (tid < kBins) {
        const uint32_t d = tid;
        uint32_t excl = 0;
        if (tile > 0) {
            int j = (int)tile - 1;
            uint32_t spins = 0;
            while (true) {
                uint32_t st[kLookback];
#pragma unroll
                for (int q = 0; q < kLookback; q++)
                    st[q] = (j - q >= 0) ? ld_relaxed(&status[(size_t)(j - q) * kBins + d]) : kFlagIncl;
                int used = 0;
                bool done = false, stop = false;
#pragma unroll
                for (int q = 0; q < kLookback; q++) {
                    if (!stop) {
                        const uint32_t flag = st[q] & ~kCountMask;
                        if (flag == 0u) {
                            stop = true;  // not published yet: retry from here
                        } else {
                            excl += st[q] & kCountMask;
                            used++;
                            if (flag == kFlagIncl) done = stop = true;
                        }
                    }
                }
                if (done) break;
                j -= used;
                // predecessors always publish (they took their tickets earlier and
                // never wait before publishing); never hang the GPU on a bug
                if (used == 0 && ++spins > (1u << 26)) __trap();
            }
            st_relaxed(&status[(size_t)tile * kBins + d], kFlagIncl | (excl + s_count[d]));
        }
        s_gofs[d] = __ldg(&bucket_base[d]) + excl;
    } else if (warp == kBins / 32) {
        constexpr int PER = kBins / 32;
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
    // global slot of tile position i with digit d = s_gofs[d] + i; warp scatter
    // offset = tile start of d + earlier warps' count of d
    if (tid < kBins) s_gofs[tid] -= s_start[tid];
    for (int i = tid; i < WARPS * kBins; i += kSortBlock) s_off[i] += s_start[i & (kBins - 1)];
    __syncthreads();

    // ---- scatter into shared memory in digit order
    const uint32_t *off = s_off + warp * kBins;
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        const uint32_t idx = wbase + it * 32u + lane;
        if (idx < tile_n) {
            const uint32_t r = (it & 1) ? (rank2[it / 2] >> 16) : (rank2[it / 2] & 0xffffu);
            const uint32_t pos = off[digit8(v[it], shift)] + r;
            s_k[pos] = v[it];
            if constexpr (KV) s_vout[pos] = s_vin[idx];
        }
    }
    __syncthreads();

    // ---- write out: consecutive tile slots of one digit -> consecutive global slots
#pragma unroll 4
    for (uint32_t i = tid; i < tile_n; i += kSortBlock) {
        const uint32_t x = s_k[i];
        const uint32_t o = s_gofs[digit8(x, shift)] + i;
        keys_out[o] = (x + out_add) ^ out_flip;
        if constexpr (KV) vals_out[o] = s_vout[i];
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
