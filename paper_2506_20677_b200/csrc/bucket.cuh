// bucket.cuh — K10: stable in-shared-memory LSD radix sort of many independent
// segments, one CTA of BLOCK (128 or 256) threads per segment of up to BLOCK x IPT keys.  It serves
// the medium segments of ahs_sort_segments (NEXT-4: the paper's small-n path,
// Listing 1, batched) and the bucket pass of the bucket-local GENERAL
// plan (after two LSD passes over the feature-bin digits every bin is
// a contiguous bucket, and each bucket still needs sorting by its low bits).
//
// Per CTA (segment [lo, hi), len <= CAP = BLOCK IPT):
//   load      the keys (v = (key ^ flip) - sub: the ordered image, range-reduced
//             by the bucket-local plan's minimum, 0 for ahs_sort_segments) and values straight into
//             registers: warp w owns the contiguous slice [w C, (w + 1) C), C = a
//             multiple of 32 >= len / 8, lane l holds its items k at w C + 32 k + l
//             (so register order (warp, item, lane) is index order);
//   digits    the OR of key ^ first key over the segment: only the 8-bit digits in
//             which some key differs get a pass (a stable pass over a constant digit
//             is the identity);
//   per pass  count (one shared atomic per key into the warp's 256-entry table;
//             for every pass after the first it is taken right after the previous
//             pass's reload) | barrier | the 256 scan threads turn the 8 warp tables
//             into slots: digit start (block scan of the totals) + earlier warps'
//             counts | barrier | rank (one shared atomic with return per key: the
//             ordered ranking, the device's lane order being self-tested as for K6)
//             and scatter into the segment buffer | barrier | reload the registers
//             in (warp, item, lane) order.  Four shared operations per key, three
//             barriers; one buffer (the keys live in registers across the scatter);
//   store     from the registers, coalesced, output transform fused.
// Stable: every pass ranks in index order.  kout may alias kin.  A segment longer
// than CAP (or reaching past n) is counted in *bad and left as is.
#pragma once

#include "common.cuh"

namespace ahs {

template <typename K, bool KV, int IPT, int BLOCK = 256>
struct BucketSort {
    static_assert(BLOCK == 128 || BLOCK == 256, "128 or 256 threads per segment");
    static constexpr int kCap = BLOCK * IPT;
    static constexpr int kWarps = BLOCK / 32;
    // 32-bit keys with values: one 64-bit slot per pair (one scatter store and one reload per pair)
    static constexpr bool kPack = KV && sizeof(K) == 4;
    static constexpr size_t kSmem = (size_t)kCap * sizeof(K) + (KV ? (size_t)kCap * 4 : 0) +
                                    (size_t)kWarps * 256 * 4 + 256 * 4 + 64;
};

// group: segment j is [offsets[j group], offsets[min((j + 1) group, nseg)]) -- several consecutive
// buckets sorted as one (the bucket-local plan: the array is already ordered by bucket, so sorting
// a run of buckets by the whole key keeps their order); nseg counts offsets - 1 entries.
template <typename K, bool KV, int IPT, int MINB, int BLOCK>
__global__ void __launch_bounds__(BLOCK, MINB)
    k_bucket_sort(const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
                  uint32_t *__restrict__ vout, const uint32_t *__restrict__ offsets, uint32_t nseg, uint64_t n,
                  K flip, K sub, uint32_t *__restrict__ bad, const uint32_t *__restrict__ gate, uint32_t group)
{
    using C = BucketSort<K, KV, IPT, BLOCK>;
    constexpr int NW = C::kWarps, CAP = C::kCap;
    pdl_begin();
    if (gate && __ldcg(gate) == 0u) return;
    extern __shared__ __align__(16) uint8_t bk_smem[];
    K *const kb = reinterpret_cast<K *>(bk_smem);
    [[maybe_unused]] uint32_t *const vb = reinterpret_cast<uint32_t *>(bk_smem + (size_t)CAP * sizeof(K));
    [[maybe_unused]] uint64_t *const pb = reinterpret_cast<uint64_t *>(bk_smem);  // kPack: (value << 32) | key
    uint32_t *const tab = reinterpret_cast<uint32_t *>(bk_smem + (size_t)CAP * sizeof(K) +
                                                       (KV ? (size_t)CAP * 4 : 0));  // [NW][256]
    uint32_t *const s_wsum = tab + NW * 256;                                          // [8]
    __shared__ uint32_t s_diff[2];

    const uint64_t s0 = (uint64_t)blockIdx.x * group;
    if (s0 >= nseg) return;
    const uint32_t lo = __ldg(&offsets[s0]), hi = __ldg(&offsets[min(s0 + group, (uint64_t)nseg)]);
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    if (hi < lo || (uint64_t)hi > n || hi - lo > (uint32_t)CAP) {
        if (t == 0) atomicAdd(bad, 1u);
        return;
    }
    const uint32_t len = hi - lo;
    if (len < 2) {
        if (len == 1 && t == 0 && kout != kin) {
            kout[lo] = kin[lo];
            if constexpr (KV) vout[lo] = vin[lo];
        }
        return;
    }
    // warp slices: C keys each (a multiple of 32), the last ones possibly short or empty
    const uint32_t Cw = ((len + NW - 1) / NW + 31u) & ~31u;
    const uint32_t wb = min(len, warp * Cw), we = min(len, wb + Cw);
    auto slot = [&](int k) { return wb + (uint32_t)k * 32u + lane; };
    auto valid = [&](int k) { return slot(k) < we; };

    if (t == 0) s_diff[0] = s_diff[1] = 0u;
    for (int i = t; i < NW * 256; i += BLOCK) tab[i] = 0u;
    __syncthreads();
    const K first = (K)((kin[lo] ^ flip) - sub);
    K x[IPT];
    [[maybe_unused]] uint32_t y[KV ? IPT : 1];
    K dacc = 0;
#pragma unroll
    for (int k = 0; k < IPT; k++) {
        x[k] = valid(k) ? (K)((kin[lo + slot(k)] ^ flip) - sub) : first;
        if constexpr (KV) y[k] = valid(k) ? vin[lo + slot(k)] : 0u;
        dacc |= x[k] ^ first;
    }
    {
        const uint32_t dlo = __reduce_or_sync(kFull, (uint32_t)dacc);
        const uint32_t dhi = sizeof(K) == 8 ? __reduce_or_sync(kFull, (uint32_t)((uint64_t)dacc >> 32)) : 0u;
        if (lane == 0) {
            if (dlo) atomicOr(&s_diff[0], dlo);
            if (dhi) atomicOr(&s_diff[1], dhi);
        }
    }
    __syncthreads();
    const uint64_t diff = ((uint64_t)s_diff[1] << 32) | s_diff[0];
    uint32_t *const wt = tab + warp * 256;

    // the digits some key of the segment differs in (a stable pass over a constant digit is the identity)
    uint32_t act = 0;
#pragma unroll
    for (int b = 0; b < (int)sizeof(K); b++) act |= (((diff >> (8 * b)) & 0xffu) != 0 ? 1u : 0u) << b;
    // slots: digit start (block scan of the totals) + earlier warps' counts; thread t owns digits
    // t DPT .. t DPT + DPT - 1
    auto scan_tables = [&] {
        constexpr int DPT = 256 / BLOCK;
        uint32_t c[DPT][NW], tot = 0;
#pragma unroll
        for (int j = 0; j < DPT; j++)
#pragma unroll
            for (int w = 0; w < NW; w++) {
                c[j][w] = tab[w * 256 + t * DPT + j];
                tot += c[j][w];
            }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFull, incl, o);
            if (lane >= (uint32_t)o) incl += v;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        uint32_t run = incl - tot;
#pragma unroll
        for (int w = 0; w < NW; w++)
            if (w < (int)warp) run += s_wsum[w];
#pragma unroll
        for (int j = 0; j < DPT; j++)
#pragma unroll
            for (int w = 0; w < NW; w++) {
                tab[w * 256 + t * DPT + j] = run;
                run += c[j][w];
            }
    };

    if constexpr (C::kPack) {
        if ((diff >> 16) == 0u) {
            // Narrow segment (every key shares bits 16.. of v with the first; the bucket-local plan's
            // buckets when the feature shift is <= 16): one 32-bit slot per pair, (v & 0xffff) << 16 |
            // local index, sorted by its top half, the values parked in shared memory at their local
            // index and gathered once at the end -- the 64-bit slot scatter and reload of every pair
            // and sub-pass become 32-bit ones
            uint32_t *const ws = reinterpret_cast<uint32_t *>(bk_smem);  // [CAP] slots
            uint32_t *const vs = ws + CAP;                                 // [CAP] values by local index
            uint32_t w[IPT];
#pragma unroll
            for (int k = 0; k < IPT; k++) {
                if (valid(k)) vs[slot(k)] = y[k];
                w[k] = (((uint32_t)x[k] & 0xffffu) << 16) | slot(k);
            }
            auto wcount = [&](uint32_t sh) {
#pragma unroll
                for (int k = 0; k < IPT; k++)
                    if (valid(k)) atomicAdd(&wt[(w[k] >> sh) & 0xffu], 1u);
            };
            uint32_t wact = act & 3u;  // digits 0 and 1 of v: bits 16-23 and 24-31 of the slot
            if (wact) wcount(16u + 8u * (uint32_t)(__ffs(wact) - 1));
            while (wact) {
                const uint32_t sh = 16u + 8u * (uint32_t)(__ffs(wact) - 1);
                wact &= wact - 1u;
                __syncthreads();  // every warp's counts of this digit are in
                scan_tables();
                __syncthreads();
#pragma unroll
                for (int k = 0; k < IPT; k++) {
                    if (valid(k)) {
                        const uint32_t pos = atomicAdd(&wt[(w[k] >> sh) & 0xffu], 1u);
                        ws[pos] = w[k];
                    }
                    __syncwarp();
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < IPT; k++)
                    if (valid(k)) w[k] = ws[slot(k)];
                if (wact) {
                    for (int i = lane; i < 256; i += 32) wt[i] = 0u;
                    __syncwarp();
                    wcount(16u + 8u * (uint32_t)(__ffs(wact) - 1));
                }
            }
            __syncthreads();  // the parked values are visible (also when no digit varies)
            const uint32_t top = (uint32_t)first & 0xffff0000u;  // the bits of v every key shares
#pragma unroll
            for (int k = 0; k < IPT; k++) {
                if (valid(k)) {
                    kout[lo + slot(k)] = (K)((top | (w[k] >> 16)) + sub) ^ flip;
                    vout[lo + slot(k)] = vs[w[k] & 0xffffu];
                }
            }
            return;
        }
    }
    auto count = [&](uint32_t sh) {  // non-returning atomics: same-word lanes merge
#pragma unroll
        for (int k = 0; k < IPT; k++)
            if (valid(k)) atomicAdd(&wt[(uint32_t)(x[k] >> sh) & 0xffu], 1u);
    };
    if (act) count(8u * (uint32_t)(__ffs(act) - 1));
    while (act) {
        const uint32_t sh = 8u * (uint32_t)(__ffs(act) - 1);
        act &= act - 1u;
        auto dig = [&](K v) { return (uint32_t)(v >> sh) & 0xffu; };
        __syncthreads();  // every warp's counts of this digit are in
        scan_tables();
        __syncthreads();
        // ---- rank (lanes of one instruction served in lane order: self-tested) and scatter
#pragma unroll
        for (int k = 0; k < IPT; k++) {
            if (valid(k)) {
                const uint32_t pos = atomicAdd(&wt[dig(x[k])], 1u);
                if constexpr (C::kPack) {
                    pb[pos] = ((uint64_t)y[k] << 32) | (uint32_t)x[k];
                } else {
                    kb[pos] = x[k];
                    if constexpr (KV) vb[pos] = y[k];
                }
            }
            __syncwarp();
        }
        __syncthreads();
        // ---- reload in index order; this warp's table (only this warp touches it until the
        // next barrier) is cleared and takes the counts of the next digit
#pragma unroll
        for (int k = 0; k < IPT; k++) {
            if (valid(k)) {
                if constexpr (C::kPack) {
                    const uint64_t q = pb[slot(k)];
                    x[k] = (K)(uint32_t)q;
                    y[k] = (uint32_t)(q >> 32);
                } else {
                    x[k] = kb[slot(k)];
                    if constexpr (KV) y[k] = vb[slot(k)];
                }
            }
        }
        if (act) {
            for (int i = lane; i < 256; i += 32) wt[i] = 0u;
            __syncwarp();
            count(8u * (uint32_t)(__ffs(act) - 1));
        }
    }
#pragma unroll
    for (int k = 0; k < IPT; k++) {
        if (valid(k)) {
            kout[lo + slot(k)] = (K)(x[k] + sub) ^ flip;
            if constexpr (KV) vout[lo + slot(k)] = y[k];
        }
    }
}

}  // namespace ahs
