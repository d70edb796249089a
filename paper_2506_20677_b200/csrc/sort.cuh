// sort.cuh — K4 count_fill, K5 radix_hist (K6, the onesweep pass, is in onesweep.cuh).
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
// K6 (onesweep.cuh) is a onesweep digit pass: one read + one write of the
// keys per pass, persistent CTAs, stable shared-memory ranking, decoupled
// look-back over tile statuses.
#pragma once

#include "common.cuh"
#include "features.cuh"
#include "onesweep.cuh"

namespace ahs {

// K6 launch configurations (see onesweep.cuh), measured on B200
// (tools/passbench.cu, profiles/r01_summary.md):
//   masked ranking (no assumption on atomic lane order): keys 512 x 15 (tile
//     7680, 2 CTAs/SM), pairs 512 x 9 (tile 4608, 2 CTAs/SM);
//   ordered ranking (after the lane-order self-test): keys 512 x 16 (tile
//     8192, 2 CTAs/SM), pairs 512 x 15 (tile 7680, 1 CTA/SM).
constexpr int kSortBlock = 512;
using OsKeysM = Onesweep<false, kSortBlock, 15, kRankMasked>;
using OsPairsM = Onesweep<true, kSortBlock, 9, kRankMasked>;
using OsKeysO = Onesweep<false, kSortBlock, 16, kRankOrdered>;
using OsPairsO = Onesweep<true, kSortBlock, 15, kRankOrdered>;
#define K6_KEYS_M k_onesweep<false, kSortBlock, 15, 2, kRankMasked>
#define K6_PAIRS_M k_onesweep<true, kSortBlock, 9, 2, kRankMasked>
#define K6_KEYS_O k_onesweep<false, kSortBlock, 16, 2, kRankOrdered>
#define K6_PAIRS_O k_onesweep<true, kSortBlock, 15, 1, kRankOrdered>
constexpr int kMinTile = 4608;  // smallest K6 tile: sizes the look-back status buffer
static_assert(kMinTile <= OsKeysM::kTile && kMinTile <= OsPairsM::kTile && kMinTile <= OsKeysO::kTile &&
                  kMinTile <= OsPairsO::kTile,
              "kMinTile");

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
constexpr uint32_t kPlanMagic = 0xa45c0de1u;  // plan[5] once K5 has written a plan
constexpr int kRHBlock = 1024;
constexpr int kRHChunk = 46 * 1024;  // < 3 vectors per thread (fits 227 KB with the 4 KB static digit tables)
constexpr int kRHStages = 2;
constexpr int kRHSmem = kHistBins + kRHStages * (kRHChunk + 16);

struct JointAdd {  // packed joint counter; overflow goes straight to the marginals
    uint32_t *sh, *dig0, *dig1;
    __device__ __forceinline__ void operator()(uint32_t b, uint32_t c) const
    {
        fix(atomicAdd(&sh[b >> 1], c << ((b & 1u) << 4)), b, c);
    }
    __device__ __forceinline__ void fix(uint32_t old, uint32_t b, uint32_t c) const
    {
        const uint32_t sft = (b & 1u) << 4;
        const uint32_t h = (old >> sft) & 0xffffu;
        if (h < 0x8000u && h + c >= 0x8000u) {
            atomicSub(&sh[b >> 1], 0x8000u << sft);
            atomicAdd(&dig0[b & 255u], 0x8000u);
            atomicAdd(&dig1[b >> 8], 0x8000u);
        }
    }
    __device__ __forceinline__ void add4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) const
    {
        const uint32_t o0 = atomicAdd(&sh[b0 >> 1], 1u << ((b0 & 1u) << 4));
        const uint32_t o1 = atomicAdd(&sh[b1 >> 1], 1u << ((b1 & 1u) << 4));
        const uint32_t o2 = atomicAdd(&sh[b2 >> 1], 1u << ((b2 & 1u) << 4));
        const uint32_t o3 = atomicAdd(&sh[b3 >> 1], 1u << ((b3 & 1u) << 4));
        fix(o0, b0, 1u);
        fix(o1, b1, 1u);
        fix(o2, b2, 1u);
        fix(o3, b3, 1u);
    }
};

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1)
    k_radix_hist(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip, uint32_t sub, int passes,
                 const uint32_t *__restrict__ fhist, uint32_t nb, uint32_t fshift,
                 uint32_t *__restrict__ dhist, uint32_t *__restrict__ bucket_base,
                 uint32_t *__restrict__ ticket, uint32_t *__restrict__ plan, int skip_trivial)
{
    extern __shared__ __align__(128) uint32_t sh[];
    __shared__ uint32_t s_dig[4][256];
    __shared__ __align__(8) uint64_t bars[kRHStages];
    __shared__ bool s_last;
    __shared__ uint32_t s_triv[4];
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
#pragma unroll 16
                for (uint32_t d1 = 0; d1 < 256; d1++) {
                    const uint32_t b = (d1 << 8) | t;
                    sum += (sh[b >> 1] >> ((b & 1u) << 4)) & 0xffffu;
                }
                atomicAdd(&s_dig[0][t], sum);
            } else {
#pragma unroll 16
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
        uint32_t run = incl - sum, mx = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            bucket_base[warp * 256 + lane * 8 + j] = run;
            run += c[j];
            mx = max(mx, c[j]);
        }
        // NEXT-1: a digit that every key shares makes its pass an identity
        mx = __reduce_max_sync(kFull, mx);
        if (lane == 0) s_triv[warp] = skip_trivial && (uint64_t)mx == n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // device pass plan: executed passes renumbered 0 .. m-1; plan[4] = m, plan[5] = magic
        uint32_t m = 0;
        for (int p = 0; p < passes; p++) m += s_triv[p] ? 0u : 1u;
        uint32_t e = 0;
        for (int p = 0; p < passes; p++) {
            plan[p] = s_triv[p] ? kPassSkip : ((e << 8) | m);
            e += s_triv[p] ? 0u : 1u;
        }
        plan[4] = m;
        plan[5] = kPlanMagic;
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
