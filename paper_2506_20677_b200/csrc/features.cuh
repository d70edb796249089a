// features.cuh — K1 feat_reduce, K2 feat_hist, K3 feat_finalize.
//
// PAPER.md §III.A (line 96): the state vector v = (n, k, H), k = max - min + 1,
// H = -sum_i p_i log2 p_i (also §III.H).  DESIGN.md R1 fixes the
// support of p: 2^shift-wide buckets of key - min, at most 2^16 of them
// (exact per-value entropy whenever k <= 2^16).  Descents (presortedness,
// §I line 25 / north_star) = #{i : key[i] > key[i+1]}.
//
// Data flow (no host sync until the end):
//   K1 reads the keys once: per-block (min, max, descents) -> ws partials;
//      zeroes the overflow bins and K3's barrier word.
//   K2 reads the keys again.  Every CTA re-reduces the K1 partials (min and
//      the bucket shift), privatises the histogram in shared memory, and each
//      cluster of kHistCluster CTAs merges its shared-memory histograms over
//      DSMEM into ONE partial row in global memory (plain coalesced stores, no
//      global atomics).
//   K3 (cooperative, one CTA per 1024 bins) sums the cluster rows, computes
//      H in fp64 in a fixed order (deterministic), and the exclusive scan of
//      the histogram that COUNTING reuses.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace ahs {

namespace cg = cooperative_groups;

constexpr int kReduceBlock = 256;
constexpr int kReduceUnroll = 4;
constexpr int kHistBlock = 1024;
constexpr int kHistUnroll = 2;
constexpr int kHistCluster = 4;
constexpr int kHistSmemBytes = 128 * 1024;           // 2^16 packed 16-bit counters
constexpr uint32_t kHistWords = kHistSmemBytes / 4;  // 32768
constexpr int kFinalBlock = 1024;
constexpr uint32_t kMaxBins = 1u << 16;
constexpr int kFinalGrid = (int)(kMaxBins / kFinalBlock);  // 64

// K3 control block in ws (zeroed by K1 where noted)
struct FinalCtrl {
    uint32_t barrier;       // zeroed by K1
    uint32_t pad[31];
    uint32_t chunk_tot[kFinalGrid];
    double chunk_S[kFinalGrid];
};

// ------------------------------------------------------------------ K1 ----
template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK)
    k_feat_reduce(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip,
                  Partial *__restrict__ partials, uint32_t *__restrict__ zero_words, uint32_t nzero,
                  FinalCtrl *__restrict__ fctrl)
{
    for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < nzero; i += gridDim.x * BLOCK)
        zero_words[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) fctrl->barrier = 0u;

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
//   warp w increments copy w % R; nb <= 64 additionally warp-aggregates with
//   match.any.
// Mode B (nb > 32768): 2^16 packed counters, two per 32-bit word, each a
//   15-bit count plus a guard bit.  The thread whose atomicAdd carries a half
//   across 0x8000 owns the overflow: it subtracts 0x8000 from that half and
//   adds 32768 to the global overflow bin.  The guard bit absorbs the carry,
//   so a half never spills into its neighbour while fewer than 32768
//   increments to one bin are in flight between the crossing and its
//   correction.  Bound: each thread has at most one packed atomic in flight
//   (the next one is issued after the branch on this one's return value), a
//   warp's lanes stay within two key slots of each other (every slot has warp
//   collectives), and one slot is 128 keys: <= 32 warps x 256 = 8192 < 32768.
// Both modes first merge runs of equal bins: within a thread's 4 keys, and
// across lanes whose 4 keys all fall into one bin (sorted / nearly sorted
// input would otherwise serialise 32 lanes on one address).
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
        const uint32_t sft = (b & 1u) << 4;
        const uint32_t old = atomicAdd(&sh[b >> 1], c << sft);
        const uint32_t h = (old >> sft) & 0xffffu;
        if (h < 0x8000u && h + c >= 0x8000u) {
            atomicSub(&sh[b >> 1], 0x8000u << sft);
            atomicAdd(&ovf[b], 0x8000u);
        }
    }
};

__device__ __forceinline__ void hist_vec(const HistAdd &add, uint4 x, bool act, uint32_t umin,
                                         uint32_t shift, bool aggregate)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t b0 = (x.x - umin) >> shift, b1 = (x.y - umin) >> shift;
    const uint32_t b2 = (x.z - umin) >> shift, b3 = (x.w - umin) >> shift;
    if (aggregate) {  // few bins: match.any per key slot, one atomic per distinct bin
        const uint32_t bb[4] = {b0, b1, b2, b3};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t key = act ? bb[j] : 0xffffffffu;
            const uint32_t peers = __match_any_sync(kFull, key);
            if (act && lane == (uint32_t)(__ffs(peers) - 1)) add(bb[j], (uint32_t)__popc(peers));
        }
        return;
    }
    const bool single = act && b0 == b1 && b1 == b2 && b2 == b3;
    const uint32_t pb = __shfl_up_sync(kFull, b0, 1);
    const uint32_t smask = __ballot_sync(kFull, single);
    const bool prev_single = lane > 0 && ((smask >> (lane - 1)) & 1u);
    const bool head = single && !(prev_single && pb == b0);
    const uint32_t hmask = __ballot_sync(kFull, head);
    if (head) {
        // the run covers lanes [lane, e): e = next lane that is a head or not single
        const uint32_t stop = (hmask | ~smask) & (lane == 31u ? 0u : (0xffffffffu << (lane + 1)));
        const uint32_t e = stop ? (uint32_t)(__ffs(stop) - 1) : 32u;
        add(b0, 4u * (e - lane));
    } else if (act && !single) {
        uint32_t cur = b0, c = 1;
        if (b1 == cur) c++; else { add(cur, c); cur = b1; c = 1; }
        if (b2 == cur) c++; else { add(cur, c); cur = b2; c = 1; }
        if (b3 == cur) c++; else { add(cur, c); cur = b3; c = 1; }
        add(cur, c);
    }
}

template <int BLOCK, int UNROLL, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(BLOCK, 1)
    k_feat_hist(const uint32_t *__restrict__ keys, uint64_t n, uint32_t flip,
                const Partial *__restrict__ partials, int nparts, uint32_t *__restrict__ ovf,
                uint32_t *__restrict__ parts)
{
    extern __shared__ __align__(16) uint32_t sh[];
    cg::cluster_group cluster = cg::this_cluster();
    const Partial p = reduce_partials<BLOCK>(partials, nparts);
    const Range rg = derive_range(p.mn, p.mx, 16u);
    if (rg.nb <= 1u) return;  // k = 1 (uniform for the whole grid): no histogram
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const bool packed = rg.nb > kHistWords;
    uint32_t R = 1;
    if (!packed) {
        R = kHistWords / rg.nb;
        if (R > BLOCK / 32) R = BLOCK / 32;
    }
    const uint32_t words = packed ? (rg.nb + 1u) >> 1 : R * rg.nb;
    for (uint32_t i = threadIdx.x; i < words; i += BLOCK) sh[i] = 0u;
    __syncthreads();

    const HistAdd add{sh, ovf, packed ? 0u : (warp % R) * rg.nb, packed};
    const bool aggregate = !packed && rg.nb <= 64u;
    const uint32_t umin = p.mn, shift = rg.shift;

    const VecSplit sp = vec_split(keys, n);
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    const uint4 *vp = reinterpret_cast<const uint4 *>(keys + sp.head);
    for (uint64_t vb = (uint64_t)blockIdx.x * BLOCK + warp * 32u; vb < sp.nvec; vb += stride * UNROLL) {
        uint4 x[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const uint64_t v = vb + (uint64_t)u * stride + lane;
            x[u] = v < sp.nvec ? ld_nc_v4(vp + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const uint64_t v = vb + (uint64_t)u * stride + lane;
            const uint4 y = make_uint4(x[u].x ^ flip, x[u].y ^ flip, x[u].z ^ flip, x[u].w ^ flip);
            hist_vec(add, y, v < sp.nvec, umin, shift, aggregate);
        }
    }
    if (blockIdx.x == 0 && warp == 0) {  // head / tail keys, one per lane
        const uint64_t i = lane < 3 ? lane : sp.tail0 + (lane - 3);
        const bool act = lane < 3 ? i < sp.head : (lane < 6 && i < n);
        const uint32_t u = act ? (keys[i] ^ flip) : umin;
        const uint32_t key = act ? (u - umin) >> shift : 0xffffffffu;
        const uint32_t peers = __match_any_sync(kFull, key);
        if (act && lane == (uint32_t)(__ffs(peers) - 1)) add(key, (uint32_t)__popc(peers));
    }
    __syncthreads();
    if (!packed && R > 1) {  // fold the private copies into copy 0
        for (uint32_t b = threadIdx.x; b < rg.nb; b += BLOCK) {
            uint32_t s = 0;
            for (uint32_t r = 0; r < R; r++) s += sh[r * rg.nb + b];
            sh[b] = s;
        }
    }
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
        for (uint32_t w = w0 + threadIdx.x; w < w1; w += BLOCK) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int c = 0; c < CL; c++) {
                const uint32_t v = peer[c][w];
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
// Cooperative launch of kFinalGrid CTAs x 1024 threads (co-resident by
// construction, 1 CTA per SM): CTA j owns bins [1024 j, 1024 j + 1024).
//   phase 1: c_b = sum of the cluster rows + overflow; hist[b] = c_b;
//            chunk total and chunk sum of c_b log2 c_b (fixed tree).
//   barrier (atomic counter zeroed by K1; kFinalGrid CTAs are resident)
//   phase 2: scan[b] = exclusive prefix (chunk offsets + local), scan[nb] = n;
//            CTA 0: H = log2 n - (1/n) sum_j S_j (fixed order), clamped to
//            [0, log2 nb] (R11), written with the other features.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1)
    k_feat_finalize(uint64_t n, const Partial *__restrict__ partials, int nparts,
                    const uint32_t *__restrict__ parts, int nrows, const uint32_t *__restrict__ ovf,
                    uint32_t *__restrict__ hist, uint32_t *__restrict__ scan, FinalCtrl *__restrict__ fctrl,
                    DevFeatures *__restrict__ out)
{
    const Partial p = reduce_partials<BLOCK>(partials, nparts);
    const Range rg = derive_range(p.mn, p.mx, 16u);
    __shared__ uint32_t s_cnt[BLOCK / 32];
    __shared__ double s_sum[BLOCK / 32];
    __shared__ uint32_t s_off;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t b = blockIdx.x * BLOCK + threadIdx.x;

    // ---- phase 1
    uint32_t c = 0;
    if (b < rg.nb) {
        if (rg.nb == 1u) {
            c = (uint32_t)n;
        } else {
            c = __ldcg(&ovf[b]);
            for (int r = 0; r < nrows; r++) c += __ldcg(&parts[(size_t)r * kMaxBins + b]);
        }
        hist[b] = c;
    }
    double S = c > 1u ? (double)c * log2((double)c) : 0.0;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S += __shfl_down_sync(kFull, S, o);
    if (lane == 31) s_cnt[warp] = incl;
    if (lane == 0) s_sum[warp] = S;
    __syncthreads();
    uint32_t wofs = 0;
    for (uint32_t w = 0; w < warp; w++) wofs += s_cnt[w];
    const uint32_t local_excl = wofs + incl - c;
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        double cs = 0.0;
        for (int w = 0; w < BLOCK / 32; w++) {
            tot += s_cnt[w];
            cs += s_sum[w];
        }
        fctrl->chunk_tot[blockIdx.x] = tot;
        fctrl->chunk_S[blockIdx.x] = cs;
        __threadfence();
        atomicAdd(&fctrl->barrier, 1u);
        uint32_t spins = 0;
        while (ld_relaxed(&fctrl->barrier) < gridDim.x)
            if (++spins > (1u << 28)) __trap();
        __threadfence();
        uint32_t off = 0;
        for (uint32_t j = 0; j < blockIdx.x; j++) off += __ldcg(&fctrl->chunk_tot[j]);
        s_off = off;
    }
    __syncthreads();
    // ---- phase 2
    if (b < rg.nb) scan[b] = s_off + local_excl;
    if (b == rg.nb - 1u) scan[rg.nb] = (uint32_t)n;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double tot = 0.0;
        for (int j = 0; j < (int)gridDim.x; j++) tot += __ldcg(&fctrl->chunk_S[j]);
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
