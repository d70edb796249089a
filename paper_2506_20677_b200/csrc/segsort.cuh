// segsort.cuh — K9 (NEXT-4): batched sorts of many small independent segments,
// the GPU form of the paper's small-n path (Insertion Sort for n <= 20,
// PAPER.md §III.E Listing 1; the small-n results, line 490).
// Segment s is keys[offsets[s] .. offsets[s+1]), sorted ascending and stably
// (values travel with their keys); segments are disjoint and in order.
//
//   K9s  max segment <= 32: a CTA of 256 threads owns 256 consecutive segments
//        (<= 8192 keys, one contiguous range): coalesced load of the range into
//        shared memory; each thread takes its segment into registers (padded to
//        L in {8, 16, 20, 24, 32} with the largest key) and runs Listing 1's
//        insertion sort as unrolled adjacent swaps (strict > : stable); coalesced
//        store.
//   K9m  max segment <= 2048: one CTA per segment, every segment padded to
//        P = 4 BLOCK (256 .. 2048, from the declared maximum), 4 records per
//        thread in registers: a fully unrolled bitonic network (in-register,
//        warp-shuffle and, for strides >= 128, shared-memory exchanges)
//        in shared memory on (key, original index) -- unique, so the result is
//        the stable order -- padded to a power of two with (max, max) records;
//        values gathered by the sorted indices.
// Keys compare as unsigned after `flip` (the sign bit for signed types).  A
// segment longer than the declared maximum (or reaching past n) is left as is
// and counted in *bad (device word): never an out-of-bounds access.
#pragma once

#include "common.cuh"

namespace ahs {

constexpr int kSegSmallBlock = 256;
constexpr int kSegSmallMax = 32;
constexpr int kSegMedBlock = 512;
constexpr int kSegMedMax = 2048;

template <typename K, bool KV>
constexpr size_t seg_small_smem()
{
    return (size_t)kSegSmallBlock * kSegSmallMax * (sizeof(K) + (KV ? 4 : 0));
}

template <typename K, bool KV, int L>
__global__ void __launch_bounds__(kSegSmallBlock)
    k_seg_small(const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
                uint32_t *__restrict__ vout, const uint32_t *__restrict__ offsets, uint32_t nseg, uint64_t n, K flip,
                uint32_t maxlen, uint32_t *__restrict__ bad)
{
    static_assert(L >= 2 && L <= kSegSmallMax, "register network length");
    pdl_begin();
    constexpr uint32_t CAP = kSegSmallBlock * kSegSmallMax;
    extern __shared__ __align__(16) uint8_t seg_smem[];  // keys [CAP] then values [CAP]: seg_small_smem<K, KV>()
    K *sk = reinterpret_cast<K *>(seg_smem);
    [[maybe_unused]] uint32_t *sv = reinterpret_cast<uint32_t *>(seg_smem + CAP * sizeof(K));
    __shared__ uint32_t s_ok;
    const uint32_t s0 = blockIdx.x * kSegSmallBlock, s1 = min(nseg, s0 + kSegSmallBlock);
    const uint32_t base = __ldg(&offsets[s0]), end = __ldg(&offsets[s1]);
    // the range must hold the CTA's segments (each <= L keys, inside [0, n))
    if (threadIdx.x == 0) s_ok = (end >= base && (uint64_t)end <= n && end - base <= CAP) ? 1u : 0u;
    const uint32_t my = s0 + threadIdx.x;
    uint32_t lo = 0, hi = 0;
    bool mine = my < s1;
    if (mine) {
        lo = __ldg(&offsets[my]);
        hi = __ldg(&offsets[my + 1]);
        if (hi < lo || hi - lo > maxlen || lo < base || hi > end) mine = false;  // maxlen <= L
    }
    __syncthreads();
    if (!s_ok) {
        if (my < s1) atomicAdd(bad, 1u);
        return;
    }
    if (my < s1 && !mine) atomicAdd(bad, 1u);
    const uint32_t len = end - base;
    for (uint32_t i = threadIdx.x; i < len; i += kSegSmallBlock) {
        sk[i] = kin[base + i] ^ flip;
        if constexpr (KV) sv[i] = vin[base + i];
    }
    __syncthreads();
    if (mine) {
        // the segment into registers, padded with the largest key (padding stays
        // last: the network only moves a key past a strictly greater one)
        const uint32_t a = lo - base, m = hi - lo;
        K r[L];
        [[maybe_unused]] uint32_t q[KV ? L : 1];
#pragma unroll
        for (int i = 0; i < L; i++) {
            r[i] = (uint32_t)i < m ? sk[a + i] : ~K(0);
            if constexpr (KV) q[i] = (uint32_t)i < m ? sv[a + i] : 0u;
        }
        // Listing 1 as adjacent swaps: key i moves left past every
        // strictly greater key (stable); unrolled so the array stays in registers
#pragma unroll
        for (int i = 1; i < L; i++) {
#pragma unroll
            for (int j = i; j > 0; j--) {
                const bool sw = r[j - 1] > r[j];
                const K x = r[j - 1], y = r[j];
                r[j - 1] = sw ? y : x;
                r[j] = sw ? x : y;
                if constexpr (KV) {
                    const uint32_t u = q[j - 1], w = q[j];
                    q[j - 1] = sw ? w : u;
                    q[j] = sw ? u : w;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < L; i++)
            if ((uint32_t)i < m) {
                sk[a + i] = r[i];
                if constexpr (KV) sv[a + i] = q[i];
            }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < len; i += kSegSmallBlock) {
        kout[base + i] = sk[i] ^ flip;
        if constexpr (KV) vout[base + i] = sv[i];
    }
}

// (key, index) order: unique, so a sorting network over it yields the stable order
template <typename K>
__device__ __forceinline__ bool rec_gt(K a, uint32_t ia, K b, uint32_t ib)
{
    return a > b || (a == b && ia > ib);
}

template <typename K, bool KV, int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_seg_medium(const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
                 uint32_t *__restrict__ vout, const uint32_t *__restrict__ offsets, uint32_t nseg, uint64_t n, K flip,
                 uint32_t maxlen, uint32_t *__restrict__ bad)
{
    // every segment of the launch is padded to P = 4 BLOCK records ((max key, position)
    // records sort after the real ones); thread t holds positions 4t .. 4t + 3 in registers
    constexpr int E = 4, P = BLOCK * E;
    static_assert(P <= kSegMedMax && BLOCK % 32 == 0, "segment capacity");
    pdl_begin();
    __shared__ K sk[P];
    __shared__ uint32_t si[P];
    __shared__ uint32_t sv[KV ? P : 1];  // values staged too: in place is safe
    const uint32_t seg = blockIdx.x;
    if (seg >= nseg) return;
    const uint32_t lo = __ldg(&offsets[seg]), hi = __ldg(&offsets[seg + 1]);
    if (hi < lo || (uint64_t)hi > n || hi - lo > maxlen || hi - lo > (uint32_t)P) {
        if (threadIdx.x == 0) atomicAdd(bad, 1u);
        return;
    }
    const uint32_t len = hi - lo, t = threadIdx.x;
    if (len < 2) {
        if (len == 1 && t == 0) {
            kout[lo] = kin[lo];
            if constexpr (KV) vout[lo] = vin[lo];
        }
        return;
    }
    for (uint32_t i = t; i < (uint32_t)P; i += BLOCK) {  // coalesced staging
        sk[i] = i < len ? (kin[lo + i] ^ flip) : ~K(0);
        if constexpr (KV)
            if (i < len) sv[i] = vin[lo + i];
    }
    __syncthreads();
    K key[E];
    uint32_t idx[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        key[e] = sk[t * E + e];
        idx[e] = t * E + e;
    }
    // bitonic network, fully unrolled: stride j < E in registers, j < 32 E by warp
    // shuffles (partner lane t ^ j / E), larger strides through shared memory
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < E) {
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int pe = e ^ j;
                    if (pe > e) {
                        const bool up = ((t * E + e) & k) == 0;
                        if (rec_gt(key[e], idx[e], key[pe], idx[pe]) == up) {
                            const K tk = key[e];
                            key[e] = key[pe];
                            key[pe] = tk;
                            const uint32_t ti = idx[e];
                            idx[e] = idx[pe];
                            idx[pe] = ti;
                        }
                    }
                }
            } else {
                K ok[E];
                uint32_t oi[E];
                if (j < E * 32) {
#pragma unroll
                    for (int e = 0; e < E; e++) {
                        ok[e] = __shfl_xor_sync(kFull, key[e], j / E);
                        oi[e] = __shfl_xor_sync(kFull, idx[e], j / E);
                    }
                } else {
                    __syncthreads();  // the previous exchange's reads are done
#pragma unroll
                    for (int e = 0; e < E; e++) {
                        sk[t * E + e] = key[e];
                        si[t * E + e] = idx[e];
                    }
                    __syncthreads();
#pragma unroll
                    for (int e = 0; e < E; e++) {
                        ok[e] = sk[(t * E + e) ^ j];
                        oi[e] = si[(t * E + e) ^ j];
                    }
                }
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const uint32_t p = t * E + e;
                    const bool up = (p & k) == 0, lower = (p & j) == 0;
                    // ascending: the lower position keeps the smaller record
                    const bool take = rec_gt(key[e], idx[e], ok[e], oi[e]) == (lower == up);
                    if (take) {
                        key[e] = ok[e];
                        idx[e] = oi[e];
                    }
                }
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++) {
        sk[t * E + e] = key[e];
        si[t * E + e] = idx[e];
    }
    __syncthreads();
    for (uint32_t i = t; i < len; i += BLOCK) {  // coalesced store; values by the sorted indices
        kout[lo + i] = sk[i] ^ flip;
        if constexpr (KV) vout[lo + i] = sv[si[i]];
    }
}

}  // namespace ahs
