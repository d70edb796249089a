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
#include "onesweep2.cuh"

namespace ahs {

// K6 launch configurations (see onesweep.cuh), measured on B200
// (tools/passbench.cu, profiles/r01_summary.md):
//   masked ranking (no assumption on atomic lane order): keys 512 x 15 (tile
//     7680, 2 CTAs/SM), pairs 512 x 9 (tile 4608, 2 CTAs/SM);
//   ordered ranking (after the lane-order self-test): keys 512 x 16 (tile
//     8192, 2 CTAs/SM), pairs 256 x 25 (tile 6400, 2 CTAs/SM, 110 KB of shared
//     memory each; with the packed 64-bit reorder slots 3-5 % faster than
//     384 x 16 at 2^26 / 2^28: profiles/r02_k6_shapes3.txt).
constexpr int kSortBlock = 512;
constexpr int kSortBlockPairsO = 384;  // 64-bit keys / values (ordered)
constexpr int kSortBlockPairs32O = 256;
using OsKeysM = Onesweep<false, kSortBlock, 15, kRankMasked>;
using OsPairsM = Onesweep<true, kSortBlock, 9, kRankMasked>;
using OsKeysO = Onesweep<false, kSortBlock, 16, kRankOrdered>;
using OsPairsO = Onesweep<true, kSortBlockPairs32O, 25, kRankOrdered>;
#define K6_KEYS_M k_onesweep<false, kSortBlock, 15, 2, kRankMasked>
#define K6_PAIRS_M k_onesweep<true, kSortBlock, 9, 2, kRankMasked>
#define K6_KEYS_O k_onesweep<false, kSortBlock, 16, 2, kRankOrdered>
#define K6_PAIRS_O k_onesweep<true, kSortBlockPairs32O, 25, 2, kRankOrdered>
// keys-only ordered passes over n >= kLargeN: 512 x 21 (tile 10752; 56 B of register spill at the
// 64-register cap).  In the pipeline at 2^26 (tools/quickbench.py, profiles/r02_summary.md) 512 x 18 /
// 20 / 21 / 22 sort cfg4a in 779 / 749 / 743 / 738 us and cfg4b in 765 / 724 / 730 / 746 us: fewer tiles
// mean fewer scans, look-backs and barriers per key.  (384 x 24: 1 % slower than 512 x 18 on cfg4a.)
// At 2^24 (cfg2) 512 x 16 / 18 / 20 / 22 sort in 259 / 250 / 247 / 242 us, so the shape serves n >= 2^24;
// below, 512 x 16 keeps more tiles than resident CTAs.
constexpr uint64_t kLargeN = 1ull << 24;
constexpr int kSortBlockOL = 512;
using OsKeysOL = Onesweep<false, kSortBlockOL, 21, kRankOrdered>;
#define K6_KEYS_OL k_onesweep<false, kSortBlockOL, 21, 2, kRankOrdered>
// 64-bit keys (NEXT-3), 2 CTAs/SM each: ordered keys 384 x 16 (tile 6144, 110 KB
// of shared memory; cfg6 pass 315 -> 300 us against 384 x 14), ordered pairs 384 x 10
// (3840, 108 KB; 11 % faster than 384 x 8; 384 x 11 drops to one CTA per SM: 467 -> 594 us),
// masked keys 512 x 9 (4608, 111 KB), masked pairs 512 x 5 (2560).
using OsKeys64M = Onesweep<false, kSortBlock, 9, kRankMasked, uint64_t>;
using OsPairs64M = Onesweep<true, kSortBlock, 5, kRankMasked, uint64_t>;
using OsKeys64O = Onesweep<false, kSortBlockPairsO, 16, kRankOrdered, uint64_t>;
using OsPairs64O = Onesweep<true, kSortBlockPairsO, 10, kRankOrdered, uint64_t>;
#define K6W_KEYS_M k_onesweep<false, kSortBlock, 9, 2, kRankMasked, uint64_t>
#define K6W_PAIRS_M k_onesweep<true, kSortBlock, 5, 2, kRankMasked, uint64_t>
#define K6W_KEYS_O k_onesweep<false, kSortBlockPairsO, 16, 2, kRankOrdered, uint64_t>
#define K6W_PAIRS_O k_onesweep<true, kSortBlockPairsO, 10, 2, kRankOrdered, uint64_t>
// 64-bit values (NEXT-3 payloads), 2 CTAs/SM: 32-bit keys ordered 384 x 10 (3840), masked 512 x 5
// (2560); 64-bit keys ordered 384 x 7 (2688), masked 256 x 11 (2816).
using OsPairsV64O = Onesweep<true, kSortBlockPairsO, 10, kRankOrdered, uint32_t, uint64_t>;
using OsPairsV64M = Onesweep<true, kSortBlock, 5, kRankMasked, uint32_t, uint64_t>;
using OsPairs64V64O = Onesweep<true, kSortBlockPairsO, 7, kRankOrdered, uint64_t, uint64_t>;
using OsPairs64V64M = Onesweep<true, 256, 11, kRankMasked, uint64_t, uint64_t>;
#define K6V_PAIRS_O k_onesweep<true, kSortBlockPairsO, 10, 2, kRankOrdered, uint32_t, uint64_t>
#define K6V_PAIRS_M k_onesweep<true, kSortBlock, 5, 2, kRankMasked, uint32_t, uint64_t>
#define K6WV_PAIRS_O k_onesweep<true, kSortBlockPairsO, 7, 2, kRankOrdered, uint64_t, uint64_t>
#define K6WV_PAIRS_M k_onesweep<true, 256, 11, 2, kRankMasked, uint64_t, uint64_t>
// K6 v2 (onesweep2.cuh: hot-digit ranking) for RADIX passes over 32-bit keys (ordered ranking):
// the FSM sends low-entropy inputs there, whose digits are skewed (cfg3's last pass: 64 % one
// digit).  On uniform digits it is 1-4 % slower than K6, so GENERAL keeps K6.  Keys: 512 x 22 (tile
// 11264, no spills): cfg3 sort 477 (512 x 18) -> 455 (x 20) -> 443 us (x 22); 384 x 28: 451 us.
using Os2Keys = Onesweep2<false, 512, 22, 8>;
using Os2Pairs = Onesweep2<true, kSortBlockPairsO, 16, 8>;
#define K6V2_KEYS k_onesweep2<false, 512, 22, 2, 8>
#define K6V2_PAIRS k_onesweep2<true, kSortBlockPairsO, 16, 2, 8>
// key-value COUNTING with 256 < k <= 1024 as ONE stable 10-bit scatter (opt-in: ahs_set_count_kv_single;
// the default runs two 8-bit passes, measured faster: profiles/r02_summary.md)
using Os2Pairs10 = Onesweep2<true, 256, 16, 10>;
#define K6V2_PAIRS10 k_onesweep2<true, 256, 16, 2, 10>
constexpr int kMinTile = 2560;  // smallest K6 tile: sizes the look-back status regions
static_assert(kMinTile <= OsKeysM::kTile && kMinTile <= OsPairsM::kTile && kMinTile <= OsKeysO::kTile &&
                  kMinTile <= OsKeysOL::kTile &&
                  kMinTile <= OsPairsO::kTile && kMinTile <= OsKeys64M::kTile &&
                  kMinTile <= OsPairs64M::kTile && kMinTile <= OsKeys64O::kTile && kMinTile <= OsPairs64O::kTile &&
                  kMinTile <= OsPairsV64O::kTile && kMinTile <= OsPairsV64M::kTile &&
                  kMinTile <= OsPairs64V64O::kTile && kMinTile <= OsPairs64V64M::kTile &&
                  kMinTile <= Os2Keys::kTile && kMinTile <= Os2Pairs::kTile && kMinTile <= Os2Pairs10::kTile,
              "kMinTile");

// ------------------------------------------------------------------ K5 ----
// Digit histograms of v = (key ^ flip) - min for the `passes` 8-bit digits,
// without reading the keys:
//   digits whose bits lie inside [fshift, 32) are read off the feature
//     histogram (exact counts of v >> fshift: a bucket's keys share those bits);
//   digit 0 when fshift > 0: K1's per-CTA histograms of the raw low byte,
//     rotated by min's low byte (v's low byte = raw low byte - min's, mod 256);
//   digit 1 when fshift > 8: K2's per-CTA histograms of digit 1 of v.
// (32-bit keys: fshift <= 16, so no other digit needs the keys.  64-bit keys
// (NEXT-3): digits 2 .. of v below fshift are counted from the keys by K5b,
// k_digit_count64, into dhist before K5 runs.)  Marginals are flushed with
// global atomics into dhist (zeroed by the host's memset); the last CTA turns
// them into exclusive bucket bases and writes the pass plan (NEXT-1):
// plan[p] for p < kMaxPasses, plan[kMaxPasses] = executed passes m,
// plan[kMaxPasses + 1] = kPlanMagic.
constexpr int kMaxPasses = 8;                 // 64-bit keys
constexpr uint32_t kPlanMagic = 0xa45c0de1u;  // plan[kMaxPasses + 1] once K5 has written a plan
constexpr int kPlanBL = kMaxPasses + 2;       // plan[kPlanBL] = 1: bucket-local plan (K10 runs after the passes)
constexpr int kRHBlock = 1024;
constexpr int kRowCtas = 4;  // K5 CTAs per row set (K1 low bytes, K2 digit 1)

// Bucket-local plan (GENERAL, 32-bit keys): two LSD passes over the two bytes of the
// feature bin (key - min) >> s -- digits at bit offsets s and s + 8 -- sort the keys stably by their
// bin, so every bin is a contiguous bucket (boundaries: the exclusive scan of the feature histogram);
// then K10 sorts each bucket in shared memory by its low s bits (the K9 segment sort with the bucket
// scan as offsets).  K5 chooses it when bl_cap > 0 and the largest bin holds <= bl_cap keys (the K10
// variant's capacity), and the classic full-width passes otherwise; the host launches both plans'
// kernels and the unused ones return at once (plan words kPassSkip, plan[kPlanBL] = 0).
template <int BLOCK, int MAXP = 4>
__global__ void __launch_bounds__(BLOCK, 1)
    k_radix_hist(uint64_t n, uint32_t sub, int passes, const uint32_t *__restrict__ fhist, uint32_t nb,
                 uint32_t fshift, const DevFeatures *__restrict__ dfeat, const uint32_t *__restrict__ byte0_rows,
                 const uint32_t *__restrict__ digit1_rows, uint32_t *__restrict__ dhist,
                 uint32_t *__restrict__ bucket_base, uint32_t *__restrict__ ticket, uint32_t *__restrict__ plan,
                 int skip_trivial, uint32_t bl_cap, uint32_t bl_group, uint32_t *__restrict__ maxbin,
                 const uint32_t *__restrict__ red)
{
    pdl_begin();
    static_assert(MAXP <= kMaxPasses && MAXP * 32 <= BLOCK, "one warp per pass in the final scan");
    __shared__ uint32_t s_dig[MAXP][256];
    __shared__ uint32_t s_bl[2][256];  // the bucket-local plan's two bin digits
    __shared__ bool s_last;
    __shared__ uint32_t s_triv[MAXP];
    __shared__ uint32_t s_blon;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const bool bl = bl_cap != 0u && fshift > 0u;
    // Digit placement (NEXT-1): the keys' ordered images all share their bits below lo (K1's AND / OR,
    // red = the reduced K1 record: words 4, 5), so v = key - min has lo zero low bits.  When lo is
    // not a multiple of 8 and the feature bins resolve every bit from lo up (lo >= fshift), the passes
    // take the digits at bit offsets lo, lo + 8, ... of v instead of 0, 8, ...: the same or fewer
    // passes, and dense digits (cfg3's values 2^18 apart: byte-aligned digits take every 4th value,
    // i.e. 8 of the 32 shared-memory banks; profiles/r02_summary.md).  Digits past the top bit are
    // constant (skipped), so this needs trivial-pass skipping.
    uint32_t lo = 0;
    if (red && !bl && skip_trivial) {
        const uint32_t varying = __ldcg(red + 4) ^ __ldcg(red + 5);
        const uint32_t l = varying ? (uint32_t)(__ffs(varying) - 1) : 0u;
        if ((l & 7u) != 0u && l >= fshift) lo = l;
    }
    auto off = [&](int p) { return lo + 8u * (uint32_t)p; };  // lo = 0: the byte-aligned digits
    for (int i = threadIdx.x; i < MAXP * 256; i += BLOCK) (&s_dig[0][0])[i] = 0u;
    for (int i = threadIdx.x; i < 2 * 256; i += BLOCK) (&s_bl[0][0])[i] = 0u;
    __syncthreads();
    // rows of K1 (digit 0): CTAs 0 .. kRowCtas-1; rows of K2 (digit 1): the next
    // kRowCtas (the grid has >= 2 kRowCtas); four threads per bin and CTA, each
    // summing every (4 kRowCtas)-th row: few dependent L2 round trips
    if (blockIdx.x < 2 * kRowCtas) {
        const bool d1 = blockIdx.x >= kRowCtas;
        if (lo == 0u && (d1 ? fshift > 8u : fshift > 0u)) {
            constexpr uint32_t PARTS = BLOCK / 256;
            const uint32_t t = threadIdx.x & 255u;
            const uint32_t part = (blockIdx.x % kRowCtas) * PARTS + (threadIdx.x >> 8);
            const int rows = d1 ? (int)__ldcg(&dfeat->nrows2) : (int)__ldcg(&dfeat->nparts);
            const uint32_t *rp = d1 ? digit1_rows : byte0_rows;
            uint32_t sum = 0;
#pragma unroll 8
            for (int r = (int)part; r < rows; r += PARTS * kRowCtas) sum += __ldcg(&rp[(size_t)r * 256 + t]);
            if (sum) atomicAdd(&s_dig[d1 ? 1 : 0][d1 ? t : ((t - sub) & 255u)], sum);
        }
    }
    // digits inside the feature buckets: this CTA's slice of the bins
    uint32_t mx_bin = 0;
    for (uint32_t b = blockIdx.x * BLOCK + threadIdx.x; b < nb; b += gridDim.x * BLOCK) {
        const uint32_t c = __ldg(&fhist[b]);
        if (!c) continue;
        const uint64_t base = (uint64_t)b << fshift;
#pragma unroll
        for (int p = 0; p < MAXP; p++)
            if (p < passes && off(p) >= fshift) atomicAdd(&s_dig[p][(uint32_t)(base >> off(p)) & 255u], c);
        if (bl) {
            atomicAdd(&s_bl[0][b & 255u], c);
            atomicAdd(&s_bl[1][(b >> 8) & 255u], c);
        }
    }
    // the bucket pass sorts groups of bl_group consecutive bins: the largest group must fit bl_cap
    if (bl)
        for (uint32_t g = blockIdx.x * BLOCK + threadIdx.x; (uint64_t)g * bl_group < nb; g += gridDim.x * BLOCK) {
            uint32_t c = 0;
            for (uint32_t b = g * bl_group; b < min(nb, (g + 1) * bl_group); b++) c += __ldg(&fhist[b]);
            mx_bin = max(mx_bin, c);
        }
    if (bl) {
        mx_bin = __reduce_max_sync(kFull, mx_bin);
        if (lane == 0 && mx_bin) atomicMax(maxbin, mx_bin);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += BLOCK) {
        const uint32_t v = (&s_dig[0][0])[i];
        if (v) atomicAdd(&dhist[i], v);
    }
    if (bl)
        for (int i = threadIdx.x; i < 2 * 256; i += BLOCK) {
            const uint32_t v = (&s_bl[0][0])[i];
            if (v) atomicAdd(&dhist[MAXP * 256 + i], v);
        }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) s_blon = bl && __ldcg(maxbin) <= bl_cap ? 1u : 0u;
    __syncthreads();
    const bool blon = s_blon != 0u;
    const int np = blon ? 2 : passes;  // digit histograms scanned: the bin digits or the classic ones
    if ((int)warp < np) {
        // exclusive scan of one digit histogram: lane owns 8 consecutive digits
        const uint32_t *src = dhist + (blon ? MAXP * 256 : 0) + warp * 256;
        uint32_t c[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            c[j] = __ldcg(&src[lane * 8 + j]);
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
        // device pass plan: executed passes renumbered 0 .. m-1, each with its digit's bit offset
        uint32_t m = 0;
        for (int p = 0; p < np; p++) m += s_triv[p] ? 0u : 1u;
        uint32_t e = 0;
        for (int p = 0; p < passes; p++) {
            const bool run = p < np && !s_triv[p];
            plan[p] = run ? plan_word(blon ? fshift + 8u * p : off(p), e, m) : kPassSkip;
            e += run ? 1u : 0u;
        }
        plan[kMaxPasses] = m;
        plan[kPlanBL] = blon ? 1u : 0u;
        plan[kMaxPasses + 1] = kPlanMagic;
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
    pdl_begin();
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

// ----------------------------------------------------------- K5b / K4w ----
// 64-bit keys (NEXT-3).
// K5b: digit histograms of v = (key ^ flip) - min for the digits p in [p0, p1)
// that neither the feature histogram nor the K1 / K2 rows give (bits between
// 16 and the feature bucket shift): one read of the keys, per-CTA shared
// tables, global atomics into dhist (zeroed; K5 adds the other digits and scans).
constexpr int kDC64Block = 512;
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_digit_count64(const uint64_t *__restrict__ keys, uint64_t n, uint64_t c0, int p0, int p1,
                    uint32_t *__restrict__ dhist)
{
    pdl_begin();
    __shared__ uint32_t s_dig[kMaxPasses - 2][256];
    for (int i = threadIdx.x; i < (kMaxPasses - 2) * 256; i += BLOCK) (&s_dig[0][0])[i] = 0u;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    for (uint64_t i = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += stride) {
        const uint64_t v = ld_nc(keys + i) - c0;  // (key ^ flip) - min = key - (min - flip)
        for (int p = p0; p < p1; p++) atomicAdd(&s_dig[p - 2][(uint32_t)(v >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (p1 - p0) * 256; i += BLOCK) {
        const uint32_t c = s_dig[p0 - 2 + i / 256][i % 256];
        if (c) atomicAdd(&dhist[(p0 + i / 256) * 256 + i % 256], c);
    }
}

// K4w: keys-only COUNTING for 64-bit keys: out[i] = min + v for scan[v] <= i <
// scan[v+1] (as K4; k <= k_counting, so the binary search is short).
constexpr int kFill64Block = 256;
__global__ void __launch_bounds__(kFill64Block)
    k_count_fill64(uint64_t *__restrict__ out, uint32_t n, const uint32_t *__restrict__ scan, uint32_t nb,
                   uint64_t out_flip, uint64_t out_add)
{
    pdl_begin();
    const uint32_t stride = gridDim.x * kFill64Block;
    for (uint32_t i = blockIdx.x * kFill64Block + threadIdx.x; i < n; i += stride)
        out[i] = ((uint64_t)upper_bin(scan, 0u, nb - 1u, i) + out_add) ^ out_flip;
}

}  // namespace ahs
