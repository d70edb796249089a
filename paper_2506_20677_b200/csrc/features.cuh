// features.cuh — K1 feat_reduce, K2 feat_hist, K3 feat_finalize.
//
// PAPER.md §III.A (line 96): the state vector v = (n, k, H), k = max - min + 1,
// H = -sum_i p_i log2 p_i (also §III.H).  DESIGN.md R1 fixes the
// support of p: 2^shift-wide buckets of key - min, at most 2^16 of them
// (exact per-value entropy whenever k <= 2^16).  Descents (presortedness,
// §I line 25 / north_star) = #{i : key[i] > key[i+1]}.
//
// Data flow (no host sync until the end):
//   K1 reads the keys once: per-block (min, max, descents) -> ws partials, and
//      per-block histograms of the raw low byte (radix digit 0); zeroes the
//      overflow bins and K3's ticket word.
//   K2 reads the keys again.  Every CTA re-reduces the K1 partials (min and
//      the bucket shift; CTA 0 publishes the reduced record for K3),
//      privatises the histogram in shared memory, and each cluster of
//      kHistCluster CTAs merges its shared-memory histograms over DSMEM into
//      ONE partial row in global memory (plain coalesced stores, no global
//      atomics).
//   K3 (one CTA per 256 bins, no grid barrier) sums the cluster rows and
//      computes H in fp64 in a fixed order (deterministic); the last CTA
//      writes the features.  The exclusive scan of the histogram that
//      COUNTING reuses is K3s, run by ahs_sort only for COUNTING.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace ahs {

namespace cg = cooperative_groups;

constexpr int kReduceBlock = 256;
constexpr int kReduceChunk = 24 * 1024;  // bytes per TMA chunk: 6 vectors per thread
constexpr int kReduceStages = 3;
constexpr int kReduceStageBytes = kReduceStages * (kReduceChunk + 16);
// K1's raw-low-byte histogram, one column per lane: word (byte << 5) | lane.  Lane l
// always hits bank l, so each atomic instruction is one shared-memory wavefront
// whatever the bytes (a plain 256-word table costs ~3.6 from bank collisions).
constexpr int kB0Words = 256 * 32;
constexpr int kReduceSmem = kReduceStageBytes + kB0Words * 4;
static_assert(kReduceStageBytes % 16 == 0, "lane table alignment");

// zero / fold the lane-column table (BLOCK threads; the fold rotates the lane
// per bin so a warp's 32 reads hit 32 banks)
template <int BLOCK>
__device__ __forceinline__ void b0_zero(uint32_t *t)
{
    for (int i = threadIdx.x; i < kB0Words / 4; i += BLOCK) reinterpret_cast<uint4 *>(t)[i] = make_uint4(0u, 0u, 0u, 0u);
}
template <int BLOCK>
__device__ __forceinline__ void b0_fold(const uint32_t *t, uint32_t *row)
{
    for (int b = threadIdx.x; b < 256; b += BLOCK) {
        uint32_t s = 0;
#pragma unroll 8
        for (int l = 0; l < 32; l++) s += t[(b << 5) | ((l + b) & 31)];
        row[b] = s;
    }
}
constexpr int kHistBlock = 1024;
constexpr int kHistChunk = 48 * 1024;  // 3 vectors per thread
constexpr int kHistStages = 2;
constexpr int kHistCluster = 2;
constexpr int kHistBins = 128 * 1024;                // bytes: 2^16 packed 16-bit counters
constexpr uint32_t kHistWords = kHistBins / 4;       // 32768
constexpr int kHistSmemBytes = kHistBins + kHistStages * (kHistChunk + 16);
constexpr int kFinalBins = 256;                      // K3 bins per CTA
constexpr int kFinalGroups = 16;                     // K3 row groups (threads per 4-bin quad)
constexpr int kFinalBlock = kFinalBins / 4 * kFinalGroups;
constexpr int kMaxHistRows = 80;                     // K2 clusters (rows of partial histograms)
constexpr uint32_t kMaxBins = 1u << 16;
constexpr int kFinalGrid = (int)(kMaxBins / kFinalBins);  // 256

// K3 control block in ws (zeroed by K1 where noted)
struct FinalCtrl {
    uint32_t barrier;  // K3's finished-CTA count, zeroed by K1
    uint32_t pad0;
    alignas(8) unsigned char reduced[24];  // K1's partials reduced (KeyTraits<K>::P), written by K2's CTA 0
    uint32_t pad[24];
    uint32_t chunk_tot[kFinalGrid];
    double chunk_S[kFinalGrid];
};

// ------------------------------------------------------------------ K1 ----
// Streams the aligned body through shared memory (TMA, kReduceStages chunks in
// flight per CTA); each thread folds whole uint4 vectors: min, max, and the
// descents inside the vector plus the one into the next key (next vector of
// the chunk, the chunk's extra successor vector, or the first tail key).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_feat_reduce(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip,
                  Partial *__restrict__ partials, uint32_t *__restrict__ zero_words, uint32_t nzero,
                  FinalCtrl *__restrict__ fctrl, uint32_t *__restrict__ byte0_rows)
{
    pdl_begin();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[kReduceStages];
    // histogram of the raw low byte of every key (for the radix sort: digit 0 of
    // key - min is this byte minus min's low byte, mod 256 -- no borrow -- so it
    // is known before min is); one row per CTA, no atomics across CTAs
    uint32_t *s_b0 = reinterpret_cast<uint32_t *>(smem_raw + kReduceStageBytes);  // lane columns
    b0_zero<BLOCK>(s_b0);
    __syncthreads();
    for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < nzero; i += gridDim.x * BLOCK)
        zero_words[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) fctrl->barrier = 0u;

    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const VecSplit sp = vec_split(keys, n);
    const uint4 *body = reinterpret_cast<const uint4 *>(keys + sp.head);
    uint32_t mn = 0xffffffffu, mx = 0u, desc = 0u, an = 0xffffffffu, orv = 0u;
    stream_chunks<kReduceStages, kReduceChunk>(
        body, sp.nvec, smem_raw, bars, [&](const uint4 *c, uint32_t nv, uint64_t v0) {
            for (uint32_t j = threadIdx.x; j < nv; j += BLOCK) {
                const uint4 x = c[j];
                const uint32_t a0 = x.x ^ flip, a1 = x.y ^ flip, a2 = x.z ^ flip, a3 = x.w ^ flip;
                bool has_next = true;
                uint32_t nxt;
                if (v0 + j + 1 < sp.nvec) {
                    nxt = c[j + 1].x ^ flip;  // in-chunk or the chunk's successor vector
                } else {
                    has_next = sp.tail0 < n;
                    nxt = has_next ? (keys[sp.tail0] ^ flip) : 0u;
                }
                mn = min(mn, min(min(a0, a1), min(a2, a3)));
                mx = max(mx, max(max(a0, a1), max(a2, a3)));
                an &= a0 & a1 & a2 & a3;
                orv |= a0 | a1 | a2 | a3;
                atomicAdd(&s_b0[((a0 & 255u) << 5) | lane], 1u);
                atomicAdd(&s_b0[((a1 & 255u) << 5) | lane], 1u);
                atomicAdd(&s_b0[((a2 & 255u) << 5) | lane], 1u);
                atomicAdd(&s_b0[((a3 & 255u) << 5) | lane], 1u);
                desc += (uint32_t)(a0 > a1) + (uint32_t)(a1 > a2) + (uint32_t)(a2 > a3) +
                        (uint32_t)(has_next && a3 > nxt);
            }
        });
    // unaligned head and tail (< 4 keys each): block 0, one thread each
    if (blockIdx.x == 0 && threadIdx.x < 8) {
        const uint64_t i = threadIdx.x < 4 ? threadIdx.x : sp.tail0 + (threadIdx.x - 4);
        const bool act = threadIdx.x < 4 ? i < sp.head : i < n;
        if (act) {
            const uint32_t a = keys[i] ^ flip;
            mn = min(mn, a);
            mx = max(mx, a);
            an &= a;
            orv |= a;
            atomicAdd(&s_b0[((a & 255u) << 5) | lane], 1u);
            if (i + 1 < n) desc += (uint32_t)(a > (keys[i + 1] ^ flip));
        }
    }

    __syncthreads();
    b0_fold<BLOCK>(s_b0, byte0_rows + (size_t)blockIdx.x * 256);
    __shared__ uint32_t s_mn[BLOCK / 32], s_mx[BLOCK / 32], s_d[BLOCK / 32], s_an[BLOCK / 32], s_or[BLOCK / 32];
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    desc = __reduce_add_sync(kFull, desc);
    an = __reduce_and_sync(kFull, an);
    orv = __reduce_or_sync(kFull, orv);
    if (lane == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
        s_d[warp] = desc;
        s_an[warp] = an;
        s_or[warp] = orv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial p{0xffffffffu, 0u, 0ull, 0xffffffffu, 0u};
        for (int w = 0; w < BLOCK / 32; w++) {
            p.mn = min(p.mn, s_mn[w]);
            p.mx = max(p.mx, s_mx[w]);
            p.desc += s_d[w];
            p.an &= s_an[w];
            p.orv |= s_or[w];
        }
        partials[blockIdx.x] = p;
    }
}

// 64-bit keys (NEXT-3): the same pass over uint4 vectors of two keys each
// (u = key ^ flip, flip = 2^63 for int64); head and tail are at most one key.
__device__ __forceinline__ VecSplit vec_split64(const uint64_t *p, uint64_t n)
{
    VecSplit s;
    const uint64_t mis = ((16u - ((uintptr_t)p & 15u)) & 15u) >> 3;
    s.head = mis < n ? mis : n;
    s.nvec = (n - s.head) >> 1;
    s.tail0 = s.head + 2ull * s.nvec;
    return s;
}

__device__ __forceinline__ uint64_t lo_hi(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_feat_reduce64(const uint64_t *__restrict__ keys, uint64_t n, uint64_t flip,
                    Partial64 *__restrict__ partials, uint32_t *__restrict__ zero_words, uint32_t nzero,
                    FinalCtrl *__restrict__ fctrl, uint32_t *__restrict__ byte0_rows)
{
    pdl_begin();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[kReduceStages];
    // raw low byte (digit 0 of key - min up to a rotation), lane columns as in K1
    uint32_t *s_b0 = reinterpret_cast<uint32_t *>(smem_raw + kReduceStageBytes);
    b0_zero<BLOCK>(s_b0);
    __syncthreads();
    for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < nzero; i += gridDim.x * BLOCK)
        zero_words[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) fctrl->barrier = 0u;

    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const VecSplit sp = vec_split64(keys, n);
    const uint4 *body = reinterpret_cast<const uint4 *>(keys + sp.head);
    uint64_t mn = ~0ull, mx = 0ull;
    uint32_t desc = 0u;
    stream_chunks<kReduceStages, kReduceChunk>(
        body, sp.nvec, smem_raw, bars, [&](const uint4 *c, uint32_t nv, uint64_t v0) {
            for (uint32_t j = threadIdx.x; j < nv; j += BLOCK) {
                const uint4 x = c[j];
                const uint64_t a0 = lo_hi(x.x, x.y) ^ flip, a1 = lo_hi(x.z, x.w) ^ flip;
                bool has_next = true;
                uint64_t nxt;
                if (v0 + j + 1 < sp.nvec) {
                    const uint4 y = c[j + 1];  // in-chunk or the chunk's successor vector
                    nxt = lo_hi(y.x, y.y) ^ flip;
                } else {
                    has_next = sp.tail0 < n;
                    nxt = has_next ? (keys[sp.tail0] ^ flip) : 0ull;
                }
                mn = min(mn, min(a0, a1));
                mx = max(mx, max(a0, a1));
                atomicAdd(&s_b0[((x.x & 255u) << 5) | lane], 1u);
                atomicAdd(&s_b0[((x.z & 255u) << 5) | lane], 1u);
                desc += (uint32_t)(a0 > a1) + (uint32_t)(has_next && a1 > nxt);
            }
        });
    if (blockIdx.x == 0 && threadIdx.x < 2) {  // unaligned head / tail key
        const uint64_t i = threadIdx.x == 0 ? 0ull : sp.tail0;
        const bool act = threadIdx.x == 0 ? sp.head > 0 : sp.tail0 < n;
        if (act) {
            const uint64_t a = keys[i] ^ flip;
            mn = min(mn, a);
            mx = max(mx, a);
            atomicAdd(&s_b0[(((uint32_t)a & 255u) << 5) | lane], 1u);
            if (i + 1 < n) desc += (uint32_t)(a > (keys[i + 1] ^ flip));
        }
    }
    __syncthreads();
    b0_fold<BLOCK>(s_b0, byte0_rows + (size_t)blockIdx.x * 256);
    __shared__ uint64_t s_mn[BLOCK / 32], s_mx[BLOCK / 32];
    __shared__ uint32_t s_d[BLOCK / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_down_sync(kFull, mn, o));
        mx = max(mx, __shfl_down_sync(kFull, mx, o));
    }
    desc = __reduce_add_sync(kFull, desc);
    if (lane == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
        s_d[warp] = desc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial64 p{~0ull, 0ull, 0ull};
        for (int w = 0; w < BLOCK / 32; w++) {
            p.mn = min(p.mn, s_mn[w]);
            p.mx = max(p.mx, s_mx[w]);
            p.desc += s_d[w];
        }
        partials[blockIdx.x] = p;
    }
}

// Reduce the 64-bit K1 partials inside one block (all threads get the result).
template <int BLOCK>
__device__ __forceinline__ Partial64 reduce_partials64(const Partial64 *__restrict__ partials, int nparts)
{
    __shared__ unsigned long long r_mn[BLOCK / 32], r_mx[BLOCK / 32], r_d[BLOCK / 32];
    __shared__ Partial64 r_out;
    unsigned long long mn = ~0ull, mx = 0ull, d = 0ull;
    for (int i = threadIdx.x; i < nparts; i += BLOCK) {
        mn = min(mn, (unsigned long long)__ldcg(&partials[i].mn));
        mx = max(mx, (unsigned long long)__ldcg(&partials[i].mx));
        d += __ldcg(&partials[i].desc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_down_sync(kFull, mn, o));
        mx = max(mx, __shfl_down_sync(kFull, mx, o));
        d += __shfl_down_sync(kFull, d, o);
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (lane == 0) {
        r_mn[warp] = mn;
        r_mx[warp] = mx;
        r_d[warp] = d;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial64 p{~0ull, 0ull, 0ull};
        for (int w = 0; w < BLOCK / 32; w++) {
            p.mn = min(p.mn, (uint64_t)r_mn[w]);
            p.mx = max(p.mx, (uint64_t)r_mx[w]);
            p.desc += r_d[w];
        }
        r_out = p;
    }
    __syncthreads();
    return r_out;
}

// Key-type traits for K2 / K3: partial record, its reduction, the derived range
template <typename K>
struct KeyTraits;
template <>
struct KeyTraits<uint32_t> {
    using P = Partial;
    template <int BLOCK>
    __device__ static P reduce(const P *p, int n);
    __device__ static Range64 range(const P &p)
    {
        const Range r = derive_range(p.mn, p.mx, 16u);
        return Range64{r.k, r.bits, r.shift, r.nb, 0u};
    }
};
template <>
struct KeyTraits<uint64_t> {
    using P = Partial64;
    template <int BLOCK>
    __device__ static P reduce(const P *p, int n);
    __device__ static Range64 range(const P &p) { return derive_range64(p.mn, p.mx, 16u); }
};

// Reduce the K1 partials inside one block (all threads get the result).
template <int BLOCK>
__device__ __forceinline__ Partial reduce_partials(const Partial *__restrict__ partials, int nparts)
{
    __shared__ uint32_t r_mn[BLOCK / 32], r_mx[BLOCK / 32], r_an[BLOCK / 32], r_or[BLOCK / 32];
    __shared__ unsigned long long r_d[BLOCK / 32];
    __shared__ Partial r_out;
    uint32_t mn = 0xffffffffu, mx = 0u, an = 0xffffffffu, orv = 0u;
    unsigned long long d = 0ull;
    for (int i = threadIdx.x; i < nparts; i += BLOCK) {
        const uint32_t *pw = reinterpret_cast<const uint32_t *>(partials + i);
        mn = min(mn, __ldcg(pw));
        mx = max(mx, __ldcg(pw + 1));
        d += __ldcg(reinterpret_cast<const unsigned long long *>(pw + 2));
        an &= __ldcg(pw + 4);
        orv |= __ldcg(pw + 5);
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    an = __reduce_and_sync(kFull, an);
    orv = __reduce_or_sync(kFull, orv);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_down_sync(kFull, d, o);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (lane == 0) {
        r_mn[warp] = mn;
        r_mx[warp] = mx;
        r_d[warp] = d;
        r_an[warp] = an;
        r_or[warp] = orv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial p{0xffffffffu, 0u, 0ull, 0xffffffffu, 0u};
        for (int w = 0; w < BLOCK / 32; w++) {
            p.mn = min(p.mn, r_mn[w]);
            p.mx = max(p.mx, r_mx[w]);
            p.desc += r_d[w];
            p.an &= r_an[w];
            p.orv |= r_or[w];
        }
        r_out = p;
    }
    __syncthreads();
    return r_out;
}

template <int BLOCK>
__device__ __forceinline__ Partial KeyTraits<uint32_t>::reduce(const Partial *p, int n)
{
    return reduce_partials<BLOCK>(p, n);
}
template <int BLOCK>
__device__ __forceinline__ Partial64 KeyTraits<uint64_t>::reduce(const Partial64 *p, int n)
{
    return reduce_partials64<BLOCK>(p, n);
}

// ------------------------------------------------------------------ K2 ----
// Mode C (nb <= 32768 / BLOCK): private per-thread counters, layout [bin][thread]
//   (conflict-free, no atomics).
// Mode A (64 < nb <= 32768): R = min(#warps, 32768 / nb) private 32-bit
//   copies; warp w increments copy w % R.
// Mode B (nb > 32768): 2^16 packed counters, two per 32-bit word, each a
//   15-bit count plus a guard bit.  The thread whose atomicAdd carries a half
//   across 0x8000 owns the overflow: it subtracts 0x8000 from that half and
//   adds 32768 to the global overflow bin.  The guard bit absorbs the carry,
//   so a half never spills into its neighbour while fewer than 32768
//   increments to one bin are in flight between the crossing and its
//   correction.  Bound: a thread has at most the four packed atomics of its
//   current vector in flight (add4 issues them back to back, then checks the
//   returns; the next vector's atomics come after those branches), a warp's
//   lanes stay within two key slots of each other (every slot has warp
//   collectives), and one slot is 128 keys: <= 32 warps x 256 = 8192 < 32768.
// Both modes first merge runs of equal bins: within a thread's 4 keys, and
// across lanes whose 4 keys all fall into one bin (sorted / nearly sorted
// input would otherwise serialise 32 lanes on one address).
// Mode B word of bin b: the pair word b >> 1 with its low five bits XORed with bits 5-9 (a bijection
// on the 32768 words).  Structured keys put their bins on a few banks otherwise: cfg3's 4096 values
// 2^18 apart fall 16 bins apart, i.e. on words 8 apart, i.e. on 4 of the 32 banks.
__device__ __forceinline__ uint32_t hist_word(uint32_t b)
{
    const uint32_t w = b >> 1;
    return w ^ ((w >> 5) & 31u);
}

struct HistAdd {
    uint32_t *sh, *ovf;
    uint32_t copy_base;
    bool packed;
    __device__ __forceinline__ void operator()(uint32_t b, uint32_t c) const
    {
        if (!packed) {
            atomicAdd(&sh[copy_base + b], c);
            return;
        }
        fix(atomicAdd(&sh[hist_word(b)], c << ((b & 1u) << 4)), b, c);
    }
    __device__ __forceinline__ void fix(uint32_t old, uint32_t b, uint32_t c) const
    {
        const uint32_t sft = (b & 1u) << 4;
        const uint32_t h = (old >> sft) & 0xffffu;
        if (h < 0x8000u && h + c >= 0x8000u) {
            atomicSub(&sh[hist_word(b)], 0x8000u << sft);
            atomicAdd(&ovf[b], 0x8000u);
        }
    }
    // four single increments: all atomics in flight before the first check
    __device__ __forceinline__ void add4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) const
    {
        if (!packed) {
            atomicAdd(&sh[copy_base + b0], 1u);
            atomicAdd(&sh[copy_base + b1], 1u);
            atomicAdd(&sh[copy_base + b2], 1u);
            atomicAdd(&sh[copy_base + b3], 1u);
            return;
        }
        const uint32_t o0 = atomicAdd(&sh[hist_word(b0)], 1u << ((b0 & 1u) << 4));
        const uint32_t o1 = atomicAdd(&sh[hist_word(b1)], 1u << ((b1 & 1u) << 4));
        const uint32_t o2 = atomicAdd(&sh[hist_word(b2)], 1u << ((b2 & 1u) << 4));
        const uint32_t o3 = atomicAdd(&sh[hist_word(b3)], 1u << ((b3 & 1u) << 4));
        // a +1 crosses 0x8000 only from 0x7fff: one combined test, the rare fix-ups behind it
        const bool f0 = ((o0 >> ((b0 & 1u) << 4)) & 0xffffu) == 0x7fffu;
        const bool f1 = ((o1 >> ((b1 & 1u) << 4)) & 0xffffu) == 0x7fffu;
        const bool f2 = ((o2 >> ((b2 & 1u) << 4)) & 0xffffu) == 0x7fffu;
        const bool f3 = ((o3 >> ((b3 & 1u) << 4)) & 0xffffu) == 0x7fffu;
        if (f0 | f1 | f2 | f3) {
            if (f0) carry(b0);
            if (f1) carry(b1);
            if (f2) carry(b2);
            if (f3) carry(b3);
        }
    }
    // move 0x8000 of bin b's packed counter into its overflow word
    __device__ __forceinline__ void carry(uint32_t b) const
    {
        atomicSub(&sh[hist_word(b)], 0x8000u << ((b & 1u) << 4));
        atomicAdd(&ovf[b], 0x8000u);
    }
};

// x holds 4 keys already mapped to v = key - min (mod 2^32); bins v >> shift.
template <typename Add>
__device__ __forceinline__ void hist_vec(const Add &add, uint4 x, bool act, uint32_t shift)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t b0 = x.x >> shift, b1 = x.y >> shift, b2 = x.z >> shift, b3 = x.w >> shift;
    const bool single = act && b0 == b1 && b1 == b2 && b2 == b3;
    const uint32_t smask = __ballot_sync(kFull, single);
    if (smask == 0u) {  // no lane with a one-bin vector: plain per-key adds (random data)
        if (act) add.add4(b0, b1, b2, b3);
        return;
    }
    const uint32_t pb = __shfl_up_sync(kFull, b0, 1);
    const bool prev_single = lane > 0 && ((smask >> (lane - 1)) & 1u);
    const bool head = single && !(prev_single && pb == b0);
    const uint32_t hmask = __ballot_sync(kFull, head);
    if (head) {
        // the run covers lanes [lane, e): e = next lane that is a head or not single
        const uint32_t stop = (hmask | ~smask) & (lane == 31u ? 0u : (0xffffffffu << (lane + 1)));
        const uint32_t e = stop ? (uint32_t)(__ffs(stop) - 1) : 32u;
        add(b0, 4u * (e - lane));
    } else if (act && !single) {
        // a vector that straddles bins (or holds an outlier of a nearly sorted run): its four
        // atomics back to back (merging its equal neighbours here cost more instructions than it
        // saved: up to four dependent atomic-and-check sequences, serialised across the lanes)
        add.add4(b0, b1, b2, b3);
    }
}

// nb <= 32768 / BLOCK: per-thread private counters, layout [bin][thread] (conflict-free,
// no atomics; the same thread's updates are ordered)
template <int BLOCK>
struct ThreadCols {
    uint32_t *sh;
    __device__ __forceinline__ void operator()(uint32_t b, uint32_t c) const
    {
        sh[b * BLOCK + threadIdx.x] += c;
    }
    __device__ __forceinline__ void add4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) const
    {
        (*this)(b0, 1u);
        (*this)(b1, 1u);
        (*this)(b2, 1u);
        (*this)(b3, 1u);
    }
};

// K: uint32_t, or uint64_t for 64-bit keys (NEXT-3: two keys per uint4, bins
// (key - min) >> shift with shift <= 48)
template <int BLOCK, int CL, typename K = uint32_t>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(BLOCK, 1)
    k_feat_hist(const K *__restrict__ keys, uint64_t n, K flip,
                const typename KeyTraits<K>::P *__restrict__ partials, int nparts, uint32_t *__restrict__ ovf,
                uint32_t *__restrict__ parts, uint32_t *__restrict__ digit1_rows, FinalCtrl *__restrict__ fctrl)
{
    pdl_begin();
    extern __shared__ __align__(128) uint32_t sh[];
    __shared__ __align__(8) uint64_t bars[kHistStages];
    cg::cluster_group cluster = cg::this_cluster();
    const auto p = KeyTraits<K>::template reduce<BLOCK>(partials, nparts);
    using P = typename KeyTraits<K>::P;
    static_assert(sizeof(P) <= sizeof(fctrl->reduced), "reduced partial");
    if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<P *>(fctrl->reduced) = p;  // for K3
    const Range64 rg = KeyTraits<K>::range(p);
    if (rg.nb <= 1u) return;  // k = 1 (uniform for the whole grid): no histogram
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const bool packed = rg.nb > kHistWords;
    const bool cols = rg.nb <= kHistWords / BLOCK;  // per-thread columns (64 bins at 512 threads)
    uint32_t R = 1;
    if (!packed && !cols) {
        R = kHistWords / rg.nb;
        if (R > BLOCK / 32) R = BLOCK / 32;
    }
    // packed: every word (hist_word's XOR can move a pair past (nb + 1) / 2)
    const uint32_t words = packed ? kHistWords : (cols ? rg.nb * BLOCK : R * rg.nb);
    for (uint32_t i = threadIdx.x; i < words; i += BLOCK) sh[i] = 0u;
    // Digit 1 of v = key - min for the radix sort, counted here when the feature
    // buckets are coarser than 2^8 (shift > 8, always the packed mode) and the
    // histogram can therefore not supply it; one row per CTA.
    __shared__ uint32_t s_d1[256];
    const bool cnt1 = rg.shift > 8u;
    for (int i = threadIdx.x; i < 256; i += BLOCK) s_d1[i] = 0u;
    __syncthreads();

    const uint32_t shift = rg.shift;
    const K c0 = (K)p.mn - flip;  // (key ^ flip) - umin == key - (umin - flip)  (mod 2^32 / 2^64)
    VecSplit sp;
    if constexpr (sizeof(K) == 4) sp = vec_split(keys, n);
    else sp = vec_split64(keys, n);
    const uint4 *body = reinterpret_cast<const uint4 *>(keys + sp.head);
    uint8_t *stage = reinterpret_cast<uint8_t *>(sh) + kHistBins;
    auto run = [&](const auto &add) {
        stream_chunks<kHistStages, kHistChunk, true>(body, sp.nvec, stage, bars,
                                               [&](const uint4 *c, uint32_t nv, uint64_t) {
            if constexpr (sizeof(K) == 4) {
            for (uint32_t j0 = 0; j0 < nv; j0 += BLOCK) {  // block-uniform trip count
                const uint32_t j = j0 + threadIdx.x;
                const bool act = j < nv;
                const uint4 x = act ? c[j] : make_uint4(c0, c0, c0, c0);
                const uint4 v = make_uint4(x.x - c0, x.y - c0, x.z - c0, x.w - c0);
                if (cnt1 && act) {
                    atomicAdd(&s_d1[(v.x >> 8) & 255u], 1u);
                    atomicAdd(&s_d1[(v.y >> 8) & 255u], 1u);
                    atomicAdd(&s_d1[(v.z >> 8) & 255u], 1u);
                    atomicAdd(&s_d1[(v.w >> 8) & 255u], 1u);
                }
                hist_vec(add, v, act, shift);
            }
            } else {
            // 64-bit keys: a thread takes two consecutive vectors (4 keys), bins computed here
            for (uint32_t j0 = 0; j0 < nv; j0 += 2 * BLOCK) {  // block-uniform trip count
                const uint32_t j = j0 + 2 * threadIdx.x;
                const bool a0 = j < nv, a1 = j + 1 < nv;
                const uint4 x = a0 ? c[j] : make_uint4(0u, 0u, 0u, 0u);
                const uint4 y = a1 ? c[j + 1] : make_uint4(0u, 0u, 0u, 0u);
                const uint64_t v0 = lo_hi(x.x, x.y) - c0, v1 = lo_hi(x.z, x.w) - c0;
                const uint64_t v2 = lo_hi(y.x, y.y) - c0, v3 = lo_hi(y.z, y.w) - c0;
                if (cnt1) {
                    if (a0) {
                        atomicAdd(&s_d1[(uint32_t)(v0 >> 8) & 255u], 1u);
                        atomicAdd(&s_d1[(uint32_t)(v1 >> 8) & 255u], 1u);
                    }
                    if (a1) {
                        atomicAdd(&s_d1[(uint32_t)(v2 >> 8) & 255u], 1u);
                        atomicAdd(&s_d1[(uint32_t)(v3 >> 8) & 255u], 1u);
                    }
                }
                const uint4 bq = make_uint4((uint32_t)(v0 >> shift), (uint32_t)(v1 >> shift),
                                            (uint32_t)(v2 >> shift), (uint32_t)(v3 >> shift));
                hist_vec(add, bq, a0 && a1, 0u);
                if (a0 && !a1) {  // the chunk's odd last vector
                    add(bq.x, 1u);
                    add(bq.y, 1u);
                }
            }
            }
        });
        if (blockIdx.x == 0 && warp == 0) {  // head / tail keys, one per lane
            const uint64_t i = lane < 3 ? lane : sp.tail0 + (lane - 3);
            if (lane < 3 ? i < sp.head : (lane < 6 && i < n)) {
                add((uint32_t)((keys[i] - c0) >> shift), 1u);
                if (cnt1) atomicAdd(&s_d1[(uint32_t)((keys[i] - c0) >> 8) & 255u], 1u);
            }
        }
    };
    if (cols) {
        run(ThreadCols<BLOCK>{sh});
    } else {
        run(HistAdd{sh, ovf, (warp % R) * rg.nb, packed});
    }
    __syncthreads();
    if (cols) {  // fold the per-thread columns: warp w sums bins w, w + 16, ...
        for (uint32_t b = warp; b < rg.nb; b += BLOCK / 32) {
            uint32_t s = 0;
            for (uint32_t t = lane; t < BLOCK; t += 32) s += sh[b * BLOCK + t];
            s = __reduce_add_sync(kFull, s);
            if (lane == 0) sh[rg.nb * BLOCK + b] = s;  // scratch past the columns (stage area is idle)
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < rg.nb; b += BLOCK) sh[b] = sh[rg.nb * BLOCK + b];
        __syncthreads();
    } else if (!packed && R > 1) {  // fold the private copies into copy 0
        for (uint32_t b = threadIdx.x; b < rg.nb; b += BLOCK) {
            uint32_t s = 0;
            for (uint32_t r = 0; r < R; r++) s += sh[r * rg.nb + b];
            sh[b] = s;
        }
    }
    if (cnt1)
        for (int i = threadIdx.x; i < 256; i += BLOCK) digit1_rows[(size_t)blockIdx.x * 256 + i] = s_d1[i];
    // merge the cluster's histograms over DSMEM: CTA rank r owns a slice
    cluster.sync();
    const uint32_t rank = cluster.block_rank();
    uint32_t *row = parts + (size_t)(blockIdx.x / CL) * kMaxBins;
    const uint32_t *peer[CL];
#pragma unroll
    for (int c = 0; c < CL; c++) peer[c] = cluster.map_shared_rank(sh, c);
    if (!packed) {
        const uint32_t per = (rg.nb + CL - 1) / CL;
        const uint32_t b0 = rank * per, b1 = min(rg.nb, b0 + per);
#pragma unroll 4
        for (uint32_t b = b0 + threadIdx.x; b < b1; b += BLOCK) {
            uint32_t s = 0;
#pragma unroll
            for (int c = 0; c < CL; c++) s += peer[c][b];
            row[b] = s;
        }
    } else {
        const uint32_t nw = (rg.nb + 1u) >> 1;
        const uint32_t per = (nw + CL - 1) / CL;
        const uint32_t w0 = rank * per, w1 = min(nw, w0 + per);
#pragma unroll 8
        for (uint32_t w = w0 + threadIdx.x; w < w1; w += BLOCK) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int c = 0; c < CL; c++) {
                const uint32_t v = peer[c][w ^ ((w >> 5) & 31u)];  // hist_word of bins 2w, 2w + 1
                lo += v & 0xffffu;
                hi += v >> 16;
            }
            row[2 * w] = lo;
            if (2 * w + 1 < rg.nb) row[2 * w + 1] = hi;
        }
    }
    cluster.sync();  // keep shared memory alive until every peer has read it
}

// ------------------------------------------------------------------ K3 ----
// kFinalGrid CTAs x kFinalBlock threads; CTA j owns bins [j * BINS, (j + 1) * BINS).
// min / max / descents come reduced from K2 (its CTA 0 publishes K1's partials
// reduced in FinalCtrl), so the row loads start after one dependent read.
// Thread (g, q) sums 16-byte quads of bins 4q .. 4q + 3 over the cluster rows
// r = g, g + GROUPS, ... (<= kMaxHistRows / GROUPS loads, all in flight: the row
// sums are latency bound), then the GROUPS partial sums of a bin meet in shared
// memory.  CTAs past the last bin (nb < 2^16) return at once; `active` remain.
//   c_b = sum of the cluster rows + overflow; hist[b] = c_b; per-CTA chunk
//   total and chunk sum S_j of c_b log2 c_b (fixed tree).
//   The last active CTA to finish (atomic count, zeroed by K1; no grid
//   barrier, no co-residency needed): H = log2 n - (1/n) sum_j S_j (fixed
//   order, independent of which CTA is last), clamped to [0, log2 nb]
//   (R11), written with the other features to `out` and, when
//   given, to the host-mapped `hout` (its seq word last, system-scope release).
// The exclusive scan of the histogram is K3s (k_hist_scan), run by ahs_sort
// only where COUNTING needs it.
template <int BLOCK>
__device__ __forceinline__ uint32_t block_sum_u32(uint32_t x, uint32_t *s_tmp)
{
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    x = __reduce_add_sync(kFull, x);
    if (lane == 0) s_tmp[warp] = x;
    __syncthreads();
    uint32_t t = 0;
    for (int w = 0; w < BLOCK / 32; w++) t += s_tmp[w];
    __syncthreads();
    return t;
}

template <int BLOCK>
__device__ __forceinline__ double block_sum_f64_fixed(double x, double *s_tmp)
{
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(kFull, x, o);
    if (lane == 0) s_tmp[warp] = x;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < BLOCK / 32; w++) t += s_tmp[w];
    __syncthreads();
    return t;
}

__device__ __forceinline__ void st_release_sys_u64(uint64_t *p, uint64_t v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// the record into the host's mapped buffer: seq (the word the host polls) last,
// with a system-scope release
__device__ __forceinline__ void write_host_features(DevFeatures *hout, const DevFeatures &f)
{
    uint64_t *hw = reinterpret_cast<uint64_t *>(hout);
    const uint64_t *fw = reinterpret_cast<const uint64_t *>(&f);
    constexpr int W = (int)(sizeof(DevFeatures) / 8);
#pragma unroll
    for (int w = 0; w < W - 1; w++) hw[w] = fw[w];
    st_release_sys_u64(hw + W - 1, f.seq);
}

template <int BLOCK, int GROUPS, typename K = uint32_t>
__global__ void __launch_bounds__(BLOCK, 2)
    k_feat_finalize(uint64_t n, int nparts,
                    const uint32_t *__restrict__ parts, int nrows, const uint32_t *__restrict__ ovf,
                    uint32_t *__restrict__ hist, FinalCtrl *__restrict__ fctrl, DevFeatures *__restrict__ out,
                    DevFeatures *__restrict__ hout, uint64_t seq)
{
    pdl_begin();
    constexpr uint32_t BINS = kFinalBins, QUADS = BINS / 4;
    constexpr int MAXR = (kMaxHistRows + GROUPS - 1) / GROUPS;
    static_assert(BLOCK == (int)QUADS * GROUPS && BLOCK >= (int)BINS, "K3 shape");
    // K1's partials, reduced by K2 (its CTA 0; K2 has completed: griddepcontrol.wait)
    const auto p = *reinterpret_cast<const typename KeyTraits<K>::P *>(fctrl->reduced);
    const Range64 rg = KeyTraits<K>::range(p);
    const uint32_t active = (rg.nb + BINS - 1u) / BINS;
    if (blockIdx.x >= active) return;  // no bins here (uniform per CTA)
    __shared__ uint32_t s_u[BLOCK / 32];
    __shared__ double s_d[BLOCK / 32];
    __shared__ __align__(16) uint32_t s_part[GROUPS][BINS];
    __shared__ uint32_t s_last;
    const uint32_t b = blockIdx.x * BINS + threadIdx.x;
    const uint32_t ov = (threadIdx.x < BINS && b < rg.nb && rg.nb > 1u) ? __ldcg(&ovf[b]) : 0u;  // with the rows
    {
        const uint32_t grp = threadIdx.x / QUADS, q = threadIdx.x % QUADS;
        const uint32_t b0 = blockIdx.x * BINS + 4u * q;  // row words past nb are read, never used
        uint4 acc = make_uint4(0u, 0u, 0u, 0u);
        if (b0 < rg.nb && rg.nb > 1u) {
#pragma unroll
            for (int j = 0; j < MAXR; j++) {
                const int r = (int)grp + j * GROUPS;
                if (r < nrows) {
                    const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(parts + (size_t)r * kMaxBins + b0));
                    acc.x += v.x;
                    acc.y += v.y;
                    acc.z += v.z;
                    acc.w += v.w;
                }
            }
        }
        *reinterpret_cast<uint4 *>(&s_part[grp][4u * q]) = acc;
    }
    __syncthreads();
    uint32_t c = 0;
    if (threadIdx.x < BINS && b < rg.nb) {
        if (rg.nb == 1u) {
            c = (uint32_t)n;
        } else {
            c = ov;
#pragma unroll
            for (int g = 0; g < GROUPS; g++) c += s_part[g][threadIdx.x];
        }
        hist[b] = c;
    }
    const uint32_t tot = block_sum_u32<BLOCK>(c, s_u);
    const double S = block_sum_f64_fixed<BLOCK>(c > 1u ? (double)c * log2((double)c) : 0.0, s_d);
    if (threadIdx.x == 0) {
        fctrl->chunk_tot[blockIdx.x] = tot;
        fctrl->chunk_S[blockIdx.x] = S;
        __threadfence();
        s_last = atomicAdd(&fctrl->barrier, 1u) == active - 1u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const double cs = threadIdx.x < active ? __ldcg(&fctrl->chunk_S[threadIdx.x]) : 0.0;
    const double tot_S = block_sum_f64_fixed<BLOCK>(cs, s_d);
    if (threadIdx.x == 0) {
        double H = 0.0;
        if (rg.nb > 1u) {
            const double dn = (double)n;
            H = log2(dn) - tot_S / dn;
            const double hmax = log2((double)rg.nb);
            if (H < 0.0) H = 0.0;
            if (H > hmax) H = hmax;
        }
        DevFeatures f{};
        f.umin = p.mn;
        f.umax = p.mx;
        f.descents = p.desc;
        f.k = rg.k;
        f.ksat = rg.ksat;
        f.bits = rg.bits;
        f.shift = rg.shift;
        f.nb = rg.nb;
        f.entropy = H;
        f.nparts = (uint32_t)nparts;               // K1 CTAs = rows of byte0_rows
        f.nrows2 = (uint32_t)nrows * kHistCluster;  // K2 CTAs = rows of digit1_rows
        f.seq = seq;
        *out = f;
        if (hout) write_host_features(hout, f);
    }
}

// ----------------------------------------------------------------- K3s ----
// scan[b] = exclusive prefix of hist over bins (scan[b] = n for nb <= b <= max(nb, 256)), for COUNTING.
// CTA j owns bins [j * BLOCK, (j + 1) * BLOCK); its offset is the sum of K3's
// chunk totals before it (BLOCK / kFinalBins chunks per CTA).
constexpr int kScanBlock = 1024;
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_hist_scan(const uint32_t *__restrict__ hist, const FinalCtrl *__restrict__ fctrl, uint32_t nb, uint32_t n,
                uint32_t *__restrict__ scan)
{
    pdl_begin();
    static_assert(BLOCK % kFinalBins == 0 && BLOCK >= kFinalGrid, "one chunk total per thread");
    __shared__ uint32_t s_u[BLOCK / 32];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t b = blockIdx.x * BLOCK + threadIdx.x;
    const uint32_t nchunks = blockIdx.x * (BLOCK / kFinalBins);
    const uint32_t before = threadIdx.x < nchunks ? __ldcg(&fctrl->chunk_tot[threadIdx.x]) : 0u;
    const uint32_t c = b < nb ? __ldcg(&hist[b]) : 0u;
    const uint32_t off = block_sum_u32<BLOCK>(before, s_u);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s_u[warp] = incl;
    __syncthreads();
    uint32_t wofs = 0;
    for (uint32_t w = 0; w < warp; w++) wofs += s_u[w];
    if (b < nb) scan[b] = off + wofs + incl - c;
    if (b == nb - 1u) scan[nb] = n;
    // K6 reads 257 bucket bases when it scatters COUNTING pairs with 8-bit digits, K6 v2 1024
    // with 10-bit digits (onesweep2.cuh: digit counts base[d + 1] - base[d], d < 1023)
    if (b > nb && b < 1024u) scan[b] = n;
}

}  // namespace ahs
