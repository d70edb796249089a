// features.cuh — K1 feat_reduce, K2 feat_hist, K3 feat_finalize.
//
// PAPER.md §III.A (line 96): the state vector v = (n, k, H), k = max - min + 1,
// H = -sum_i p_i log2 p_i (also §III.H).  DESIGN.md R1 fixes the
// support of p: 2^shift-wide buckets of key - min, at most 2^16 of them
// (exact per-value entropy whenever k <= 2^16).  Descents (presortedness,
// §I line 25 / north_star) = #{i : key[i] > key[i+1]}.
//
// Data flow (no host sync until the end):
//   K1 reads the keys once: per-block (min, max, descents) -> ws partials,
//      and zeroes the global histogram.
//   K2 reads the keys again: each block re-reduces the K1 partials to get
//      min and the bucket shift, privatises the histogram in shared memory,
//      flushes non-zero bins with global atomics.
//   K3 (one CTA) reduces the partials (descents), computes H in fp64 in a
//      fixed order, and the exclusive scan of the histogram for COUNTING.
#pragma once

#include "common.cuh"

namespace ahs {

constexpr int kReduceBlock = 256;
constexpr int kReduceUnroll = 4;
constexpr int kHistBlock = 1024;
constexpr int kHistUnroll = 4;
constexpr int kHistSmemBytes = 128 * 1024;           // 2^16 packed 16-bit counters
constexpr uint32_t kHistWords = kHistSmemBytes / 4;  // 32768
constexpr int kFinalBlock = 1024;
constexpr uint32_t kMaxBins = 1u << 16;

// ------------------------------------------------------------------ K1 ----
template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK)
    k_feat_reduce(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip,
                  Partial *__restrict__ partials, uint32_t *__restrict__ zero_words, uint32_t nzero)
{
    // zero the global histogram + scan for K2/K3 (stream order makes this safe)
    for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < nzero; i += gridDim.x * BLOCK)
        zero_words[i] = 0u;

    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const VecSplit sp = vec_split(keys, n);
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    const uint4 *vp = reinterpret_cast<const uint4 *>(keys + sp.head);

    uint32_t mn = 0xffffffffu, mx = 0u, desc = 0u;
    for (uint64_t vb = (uint64_t)blockIdx.x * BLOCK + warp * 32u; vb < sp.nvec; vb += stride * UNROLL) {
        uint4 x[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            uint64_t v = vb + (uint64_t)u * stride + lane;
            x[u] = v < sp.nvec ? ld_nc_v4(vp + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const uint64_t v = vb + (uint64_t)u * stride + lane;
            const bool act = v < sp.nvec;
            const uint32_t a0 = x[u].x ^ flip, a1 = x[u].y ^ flip, a2 = x[u].z ^ flip, a3 = x[u].w ^ flip;
            // the first key of the next vector lives in lane + 1 (same slot)
            uint32_t nxt = __shfl_down_sync(kFull, a0, 1);
            bool has_next = act;
            if (act && (lane == 31u || v + 1 >= sp.nvec)) {
                const uint64_t j = sp.head + 4ull * v + 4ull;
                has_next = j < n;
                if (has_next) nxt = keys[j] ^ flip;
            }
            if (act) {
                mn = min(mn, min(min(a0, a1), min(a2, a3)));
                mx = max(mx, max(max(a0, a1), max(a2, a3)));
                desc += (uint32_t)(a0 > a1) + (uint32_t)(a1 > a2) + (uint32_t)(a2 > a3) +
                        (uint32_t)(has_next && a3 > nxt);
            }
        }
    }
    // unaligned head and tail (< 4 keys each): block 0, one thread each
    if (blockIdx.x == 0 && threadIdx.x < 8) {
        const uint64_t i = threadIdx.x < 4 ? threadIdx.x : sp.tail0 + (threadIdx.x - 4);
        const bool act = threadIdx.x < 4 ? i < sp.head : i < n;
        if (act) {
            const uint32_t a = keys[i] ^ flip;
            mn = min(mn, a);
            mx = max(mx, a);
            if (i + 1 < n) desc += (uint32_t)(a > (keys[i + 1] ^ flip));
        }
    }

    // block reduction
    __shared__ uint32_t s_mn[BLOCK / 32], s_mx[BLOCK / 32], s_d[BLOCK / 32];
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    desc = __reduce_add_sync(kFull, desc);
    if (lane == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
        s_d[warp] = desc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial p{0xffffffffu, 0u, 0ull};
        for (int w = 0; w < BLOCK / 32; w++) {
            p.mn = min(p.mn, s_mn[w]);
            p.mx = max(p.mx, s_mx[w]);
            p.desc += s_d[w];
        }
        partials[blockIdx.x] = p;
    }
}

// Reduce the K1 partials inside one block (all threads get the result).
template <int BLOCK>
__device__ __forceinline__ Partial reduce_partials(const Partial *__restrict__ partials, int nparts)
{
    __shared__ uint32_t r_mn[BLOCK / 32], r_mx[BLOCK / 32];
    __shared__ unsigned long long r_d[BLOCK / 32];
    __shared__ Partial r_out;
    uint32_t mn = 0xffffffffu, mx = 0u;
    unsigned long long d = 0ull;
    for (int i = threadIdx.x; i < nparts; i += BLOCK) {
        const uint32_t *pw = reinterpret_cast<const uint32_t *>(partials + i);
        mn = min(mn, __ldcg(pw));
        mx = max(mx, __ldcg(pw + 1));
        d += __ldcg(reinterpret_cast<const unsigned long long *>(pw + 2));
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_down_sync(kFull, d, o);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (lane == 0) {
        r_mn[warp] = mn;
        r_mx[warp] = mx;
        r_d[warp] = d;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial p{0xffffffffu, 0u, 0ull};
        for (int w = 0; w < BLOCK / 32; w++) {
            p.mn = min(p.mn, r_mn[w]);
            p.mx = max(p.mx, r_mx[w]);
            p.desc += r_d[w];
        }
        r_out = p;
    }
    __syncthreads();
    return r_out;
}

// ------------------------------------------------------------------ K2 ----
// Mode A (nb <= 32768): R = min(#warps, 32768 / nb) private 32-bit copies;
//   warp w increments copy w % R.  nb <= 64: warp-aggregated with match.any.
// Mode B (nb > 32768): 2^16 packed counters, two per 32-bit word, each a
//   15-bit count plus a guard bit.  A thread whose atomicAdd returns 0x7FFF in
//   its half owns the overflow: it subtracts 0x8000 from that half and adds
//   32768 to the global bin.  The guard bit absorbs the carry, so a half
//   never spills into its neighbour as long as fewer than 32768 increments to
//   one bin are in flight between the overflow and its correction (at most
//   one per thread of the CTA: 1024).
struct HistOpA {
    uint32_t *sh;
    uint32_t umin, shift, nb, copy_base;
    bool aggregate;
    __device__ __forceinline__ void operator()(uint32_t u, bool act)
    {
        const uint32_t b = (u - umin) >> shift;
        if (aggregate) {
            const uint32_t key = act ? b : 0xffffffffu;
            const uint32_t peers = __match_any_sync(kFull, key);
            if (act && (threadIdx.x & 31u) == (uint32_t)(__ffs(peers) - 1))
                atomicAdd(&sh[copy_base + b], (uint32_t)__popc(peers));
        } else if (act) {
            atomicAdd(&sh[copy_base + b], 1u);
        }
    }
};

struct HistOpB {
    uint32_t *sh;
    uint32_t *ghist;
    uint32_t umin, shift;
    __device__ __forceinline__ void operator()(uint32_t u, bool act)
    {
        if (!act) return;
        const uint32_t b = (u - umin) >> shift;
        const uint32_t sft = (b & 1u) << 4;
        const uint32_t old = atomicAdd(&sh[b >> 1], 1u << sft);
        if (((old >> sft) & 0xffffu) == 0x7fffu) {
            atomicSub(&sh[b >> 1], 0x8000u << sft);
            atomicAdd(&ghist[b], 0x8000u);
        }
    }
};

template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK, 1)
    k_feat_hist(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip,
                const Partial *__restrict__ partials, int nparts, uint32_t *__restrict__ ghist)
{
    extern __shared__ uint32_t sh[];
    const Partial p = reduce_partials<BLOCK>(partials, nparts);
    const Range rg = derive_range(p.mn, p.mx, 16u);
    if (rg.nb <= 1u) return;  // k = 1: constant input, histogram not needed
    const uint32_t warp = threadIdx.x >> 5;

    if (rg.nb <= kHistWords) {
        uint32_t R = kHistWords / rg.nb;
        if (R > BLOCK / 32) R = BLOCK / 32;
        for (uint32_t i = threadIdx.x; i < R * rg.nb; i += BLOCK) sh[i] = 0u;
        __syncthreads();
        HistOpA op{sh, p.mn, rg.shift, rg.nb, (warp % R) * rg.nb, rg.nb <= 64u};
        for_each_key<UNROLL>(keys, n, flip, op);
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < rg.nb; b += BLOCK) {
            uint32_t s = 0;
            for (uint32_t r = 0; r < R; r++) s += sh[r * rg.nb + b];
            if (s) atomicAdd(&ghist[b], s);
        }
    } else {
        const uint32_t words = (rg.nb + 1u) >> 1;
        for (uint32_t i = threadIdx.x; i < words; i += BLOCK) sh[i] = 0u;
        __syncthreads();
        HistOpB op{sh, ghist, p.mn, rg.shift};
        for_each_key<UNROLL>(keys, n, flip, op);
        __syncthreads();
        for (uint32_t w = threadIdx.x; w < words; w += BLOCK) {
            const uint32_t v = sh[w];
            const uint32_t lo = v & 0xffffu, hi = v >> 16;
            if (lo) atomicAdd(&ghist[2u * w], lo);
            if (hi) atomicAdd(&ghist[2u * w + 1u], hi);
        }
    }
}

// ------------------------------------------------------------------ K3 ----
// One CTA.  H = log2 n - (1/n) * sum_b c_b log2 c_b  (= -sum p_b log2 p_b),
// fixed per-thread chunks + fixed reduction tree => deterministic.  Clamped
// to [0, log2 nb] (R11).  scan[b] = sum_{b' < b} c_b', scan[nb] = n.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_feat_finalize(uint64_t n, const Partial *__restrict__ partials, int nparts,
                    uint32_t *__restrict__ ghist, uint32_t *__restrict__ scan,
                    DevFeatures *__restrict__ out)
{
    const Partial p = reduce_partials<BLOCK>(partials, nparts);
    const Range rg = derive_range(p.mn, p.mx, 16u);
    __shared__ uint32_t s_cnt[BLOCK / 32];
    __shared__ double s_sum[BLOCK / 32];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;

    double S = 0.0;
    if (rg.nb == 1u) {
        if (threadIdx.x == 0) {
            ghist[0] = (uint32_t)n;
            scan[0] = 0u;
            scan[1] = (uint32_t)n;
        }
    } else {
        const uint32_t C = (rg.nb + BLOCK - 1) / BLOCK;
        const uint32_t b0 = min(rg.nb, threadIdx.x * C), b1 = min(rg.nb, b0 + C);
        uint32_t cnt = 0;
        for (uint32_t b = b0; b < b1; b++) {
            const uint32_t c = __ldcg(&ghist[b]);
            cnt += c;
            if (c > 1u) S += (double)c * log2((double)c);
        }
        // exclusive block scan of cnt
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        if (lane == 31) s_cnt[warp] = incl;
        __syncthreads();
        uint32_t wofs = 0;
        for (uint32_t w = 0; w < warp; w++) wofs += s_cnt[w];
        uint32_t run = wofs + incl - cnt;
        for (uint32_t b = b0; b < b1; b++) {
            scan[b] = run;
            run += __ldcg(&ghist[b]);
        }
        if (b0 < b1 && b1 == rg.nb) scan[rg.nb] = run;
    }
    // fixed-order reduction of S
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S += __shfl_down_sync(kFull, S, o);
    if (lane == 0) s_sum[warp] = S;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < BLOCK / 32; w++) tot += s_sum[w];
        double H = 0.0;
        if (rg.nb > 1u) {
            const double dn = (double)n;
            H = log2(dn) - tot / dn;
            const double hmax = log2((double)rg.nb);
            if (H < 0.0) H = 0.0;
            if (H > hmax) H = hmax;
        }
        DevFeatures f{};
        f.umin = p.mn;
        f.umax = p.mx;
        f.descents = p.desc;
        f.k = rg.k;
        f.bits = rg.bits;
        f.shift = rg.shift;
        f.nb = rg.nb;
        f.entropy = H;
        *out = f;
    }
}

}  // namespace ahs
