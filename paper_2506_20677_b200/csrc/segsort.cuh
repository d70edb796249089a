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
//   K9r  max segment <= 2048: one group of CAP / 16 threads per segment (one
//        warp up to 512 keys), an LSD radix sort in shared memory (below).
// Keys compare as unsigned after `flip` (the sign bit for signed types).  A
// segment longer than the declared maximum (or reaching past n) is left as is
// and counted in *bad (device word): never an out-of-bounds access.
#pragma once

#include "common.cuh"

namespace ahs {

constexpr int kSegSmallBlock = 256;
constexpr int kSegSmallMax = 32;
constexpr int kSegMedMax = 8192;  // K9r capacity (512 threads); also the bucket-local GENERAL pass, K10

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
    // staged path: the CTA's range [base, end) holds all its segments and fits the buffer
    if (threadIdx.x == 0) s_ok = (end >= base && (uint64_t)end <= n && end - base <= CAP) ? 1u : 0u;
    const uint32_t my = s0 + threadIdx.x;
    uint32_t lo = 0, hi = 0;
    bool mine = my < s1, inb = false;
    if (mine) {
        lo = __ldg(&offsets[my]);
        hi = __ldg(&offsets[my + 1]);
        inb = hi >= lo && (uint64_t)hi <= n;  // a real segment inside the keys
        if (!inb || hi - lo > maxlen) mine = false;  // maxlen <= L
    }
    __syncthreads();
    if (my < s1 && !mine) atomicAdd(bad, 1u);  // only the segments that are themselves bad
    // the segment sort of one thread, Listing 1 as adjacent swaps: key i moves
    // left past every strictly greater key (stable); unrolled so the array stays in registers
    auto sort_regs = [&](K(&r)[L], uint32_t(&q)[KV ? L : 1]) {
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
    };
    if (!s_ok) {
        // a bad segment (or non-monotone offsets) spoils the CTA's range: every good segment is
        // sorted straight from global memory; a too-long segment inside the keys is copied as is
        if (mine) {
            const uint32_t m = hi - lo;
            K r[L];
            uint32_t q[KV ? L : 1];
#pragma unroll
            for (int i = 0; i < L; i++) {
                r[i] = (uint32_t)i < m ? (K)(kin[lo + i] ^ flip) : ~K(0);
                if constexpr (KV) q[i] = (uint32_t)i < m ? vin[lo + i] : 0u;
            }
            sort_regs(r, q);
#pragma unroll
            for (int i = 0; i < L; i++)
                if ((uint32_t)i < m) {
                    kout[lo + i] = r[i] ^ flip;
                    if constexpr (KV) vout[lo + i] = q[i];
                }
        } else if (my < s1 && inb && kout != kin) {
            for (uint32_t i = lo; i < hi; i++) {
                kout[i] = kin[i];
                if constexpr (KV) vout[i] = vin[i];
            }
        }
        return;
    }
    if (mine && (lo < base || hi > end)) {  // non-monotone offsets: not inside the staged range
        mine = false;
        atomicAdd(bad, 1u);
    }
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
        uint32_t q[KV ? L : 1];
#pragma unroll
        for (int i = 0; i < L; i++) {
            r[i] = (uint32_t)i < m ? sk[a + i] : ~K(0);
            if constexpr (KV) q[i] = (uint32_t)i < m ? sv[a + i] : 0u;
        }
        sort_regs(r, q);
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

// K9r: one group per segment of <= CAP keys, staged in shared memory; LSD radix
// over 8-bit digits, skipping every digit all keys of the segment share (a
// stable pass over a constant digit is the identity).  Per pass:
//   count    warp w of the group owns the contiguous keys [w C, (w + 1) C), C = ceil(len / NW),
//            and counts their digits into its own table cnt[w][256];
//   scan     offsets in (digit, warp) order: warp w's first slot for digit d is
//            sum_{d' < d} total(d') + sum_{w' < w} cnt[w'][d];
//   scatter  warp w walks its keys in order, 32 at a time; peers with equal
//            digits take consecutive slots in lane order: the old value of a shared
//            atomicAdd when the device serves one instruction's lanes in lane order
//            (ORD, self-tested), else a peer mask from 8 ballots (one per digit bit).
// Keys and values ping-pong between two buffers; every step keeps index order
// among equal digits, so the sort is stable.
template <typename K, bool KV, int GROUP, int CAP>
constexpr size_t seg_radix_smem()  // per segment group
{
    return 2 * (size_t)CAP * sizeof(K) + (KV ? 2 * (size_t)CAP * 4 : 0) + (size_t)(GROUP / 32) * 256 * 4 + 256 * 4;
}

// a CTA of GROUP threads sorts one segment (one-warp groups use warp barriers;
// packing several one-warp segments per CTA measured no faster)
// gate (nullable): the launch does nothing unless *gate != 0 (the bucket-local plan word of K5)
template <typename K, bool KV, int GROUP, int CAP, bool ORD>
__global__ void __launch_bounds__(GROUP)
    k_seg_radix(const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
                uint32_t *__restrict__ vout, const uint32_t *__restrict__ offsets, uint32_t nseg, uint64_t n, K flip,
                K sub, uint32_t maxlen, uint32_t *__restrict__ bad, const uint32_t *__restrict__ gate)
{
    constexpr int NW = GROUP / 32;
    static_assert(CAP <= kSegMedMax && GROUP % 32 == 0 && CAP % 16 == 0, "segment capacity");
    pdl_begin();
    if (gate && __ldcg(gate) == 0u) return;
    extern __shared__ __align__(16) uint8_t seg_smem[];  // seg_radix_smem<K, KV, GROUP, CAP>()
    K *const kbuf0 = reinterpret_cast<K *>(seg_smem);
    K *const kbuf1 = kbuf0 + CAP;
    uint32_t *const cnt = reinterpret_cast<uint32_t *>(kbuf1 + CAP);  // [NW][256]
    uint32_t *const dbase = cnt + NW * 256;                          // [256]
    [[maybe_unused]] uint32_t *const vbuf0 = dbase + 256;
    [[maybe_unused]] uint32_t *const vbuf1 = vbuf0 + CAP;
    __shared__ uint32_t s_diff[2];
    __shared__ uint32_t s_idle[NW];  // ORD: the slot idle lanes' atomics go to
    auto gsync = [] {
        if constexpr (NW == 1) __syncwarp();
        else __syncthreads();
    };
    const uint32_t seg = blockIdx.x;
    if (seg >= nseg) return;
    const uint32_t lo = __ldg(&offsets[seg]), hi = __ldg(&offsets[seg + 1]);
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    if (hi < lo || (uint64_t)hi > n || hi - lo > maxlen || hi - lo > (uint32_t)CAP) {
        if (t == 0) atomicAdd(bad, 1u);
        return;
    }
    const uint32_t len = hi - lo;
    if (len < 2) {
        if (len == 1 && t == 0) {
            kout[lo] = kin[lo];
            if constexpr (KV) vout[lo] = vin[lo];
        }
        return;
    }
    // coalesced staging; the bits in which some key differs from the first
    if (t == 0) s_diff[0] = s_diff[1] = 0u;
    gsync();
    const K first = (K)((kin[lo] ^ flip) - sub);
    K dacc = 0;
    for (uint32_t i = t; i < len; i += GROUP) {
        const K x = (K)((kin[lo + i] ^ flip) - sub);
        kbuf0[i] = x;
        dacc |= x ^ first;
        if constexpr (KV) vbuf0[i] = vin[lo + i];
    }
    const uint32_t dlo = __reduce_or_sync(kFull, (uint32_t)dacc);
    const uint32_t dhi = sizeof(K) == 8 ? __reduce_or_sync(kFull, (uint32_t)((uint64_t)dacc >> 32)) : 0u;
    if (lane == 0) {
        if (dlo) atomicOr(&s_diff[0], dlo);
        if (dhi) atomicOr(&s_diff[1], dhi);
    }
    gsync();
    const uint64_t diff = ((uint64_t)s_diff[1] << 32) | s_diff[0];
    const uint32_t C = (len + NW - 1) / NW;
    const uint32_t wb = min(len, warp * C), we = min(len, wb + C);
    uint32_t *const wc = cnt + warp * 256;
    [[maybe_unused]] const uint32_t lt = (1u << lane) - 1u;
    int cur = 0;
    for (int b = 0; b < (int)sizeof(K); b++) {
        if (((diff >> (8 * b)) & 0xffu) == 0) continue;  // uniform over the group
        const uint32_t sh = 8u * b;
        const K *src = cur ? kbuf1 : kbuf0;
        K *dst = cur ? kbuf0 : kbuf1;
        for (uint32_t i = t; i < NW * 256u; i += GROUP) cnt[i] = 0u;
        gsync();
        for (uint32_t i = wb + lane; i < we; i += 32) atomicAdd(&wc[(uint32_t)(src[i] >> sh) & 0xffu], 1u);
        gsync();
        if constexpr (NW > 1) {
            for (uint32_t d = t; d < 256u; d += GROUP) {  // column prefix over the warps
                uint32_t run = 0;
#pragma unroll
                for (int w = 0; w < NW; w++) {
                    const uint32_t c = cnt[w * 256 + d];
                    cnt[w * 256 + d] = run;
                    run += c;
                }
                dbase[d] = run;
            }
            gsync();
        }
        if (warp == 0) {  // exclusive scan over the 256 digit totals, 8 per lane
            const uint32_t *tot = NW > 1 ? dbase : cnt;
            uint32_t v[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                v[j] = tot[lane * 8 + j];
                sum += v[j];
            }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(kFull, incl, o);
                if (lane >= (uint32_t)o) incl += x;
            }
            uint32_t ex = incl - sum;
            if constexpr (NW == 1) __syncwarp();  // every lane has read cnt before it is overwritten
#pragma unroll
            for (int j = 0; j < 8; j++) {
                // one warp: its table becomes the absolute slots directly
                if constexpr (NW == 1) cnt[lane * 8 + j] = ORD ? ex : 0u;
                dbase[lane * 8 + j] = ex;
                ex += v[j];
            }
        }
        gsync();
        if constexpr (ORD) {
            // the ordered ranking: shared atomics of one warp instruction on one word
            // return in lane order (self-tested per device, onesweep.cuh), so each
            // warp's table holds absolute slots and the atomic's old value is the slot
            if constexpr (NW > 1) {
                for (uint32_t d = t; d < 256u; d += GROUP) {
                    const uint32_t base = dbase[d];
#pragma unroll
                    for (int w = 0; w < NW; w++) cnt[w * 256 + d] += base;
                }
                gsync();
            }
            for (uint32_t i0 = wb; i0 < we; i0 += 32) {
                const uint32_t i = i0 + lane;
                const bool ok = i < we;
                const K x = ok ? src[i] : K(0);
                uint32_t *const a = ok ? wc + ((uint32_t)(x >> sh) & 0xffu) : s_idle + warp;  // full-warp
                const uint32_t pos = atomicAdd(a, 1u);
                if (ok) {
                    dst[pos] = x;
                    if constexpr (KV) (cur ? vbuf0 : vbuf1)[pos] = (cur ? vbuf1 : vbuf0)[i];
                }
                __syncwarp();
            }
        } else {
            for (uint32_t i0 = wb; i0 < we; i0 += 32) {  // warp-uniform trip count
                const uint32_t i = i0 + lane;
                const bool ok = i < we;
                const K x = ok ? src[i] : K(0);
                const uint32_t d = (uint32_t)(x >> sh) & 0xffu;
                uint32_t peers = __ballot_sync(kFull, ok);  // lanes with my digit: one vote per digit bit
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const uint32_t bq = __ballot_sync(kFull, (d >> q) & 1u);
                    peers &= ((d >> q) & 1u) ? bq : ~bq;
                }
                uint32_t wold = 0, pos = 0;
                if (ok) {
                    wold = wc[d];
                    pos = dbase[d] + wold + __popc(peers & lt);
                }
                __syncwarp();
                if (ok) {
                    dst[pos] = x;
                    if constexpr (KV) (cur ? vbuf0 : vbuf1)[pos] = (cur ? vbuf1 : vbuf0)[i];
                    if (lane == (uint32_t)(__ffs(peers) - 1)) wc[d] = wold + __popc(peers);
                }
                __syncwarp();
            }
        }
        gsync();
        cur ^= 1;
    }
    const K *fk = cur ? kbuf1 : kbuf0;
    [[maybe_unused]] const uint32_t *fv = cur ? vbuf1 : vbuf0;
    for (uint32_t i = t; i < len; i += GROUP) {
        kout[lo + i] = (K)(fk[i] + sub) ^ flip;
        if constexpr (KV) vout[lo + i] = fv[i];
    }
}

}  // namespace ahs
