// entropy.cuh — K8, NEXT-2: the paper-literal entropy (§III.A line
// 96, H = -sum_v p_v log2 p_v over the DISTINCT key values: reading "P" of
// SURVEY Appendix A) from a key array in which equal keys are contiguous
// (ahs_sort's output):  H = log2 n - (1/n) sum_runs c log2 c.
//
// One launch of G <= kEntMaxGrid CTAs, CTA c owning the contiguous chunk
// [c * chunk, (c + 1) * chunk), one read of the keys:
//   per warp    the chunk's w-th eighth, in steps of 32 x 16 keys (next step
//               prefetched); a run starts at i when i == 0 or key[i] != key[i-1]
//               and ends at i when i == n-1 or key[i] != key[i+1]; a warp
//               max-scan (carried between steps) gives every lane the start of
//               its first run.  Runs that start AND end inside the sub-chunk add
//               c log2 c (fp64, fixed order).  The sub-chunk's first run, when
//               it began earlier, is only measured (its length inside, and
//               whether it ends here); so is the last run when it continues.
//   per CTA     thread 0 stitches the warps' pieces: runs crossing warp
//               boundaries inside the chunk, and the chunk's own pieces -> S[c];
//               then takes a ticket (no grid barrier, no co-residency needed)
//   last CTA    the runs that cross chunk boundaries: the thread of each run's
//               origin chunk follows it forward to its end; then a fixed tree
//               over the chunk sums and those runs: H = log2 n - S / n, >= 0.
// Deterministic for a given G.  Work is independent of the run lengths.
#pragma once

#include "common.cuh"

namespace ahs {

constexpr int kEntBlock = 256;
constexpr int kEntItems = 16;
constexpr int kEntMaxGrid = 1024;

// per-chunk boundary record (global scratch)
struct RunPieces {
    uint64_t pre;       // length of the first run inside the chunk when it began earlier (0: a run starts at c0)
    uint64_t suf;       // length of the last run inside the chunk when it continues past c1 (0 otherwise)
    uint32_t pre_ends;  // that first run ends inside the chunk
    uint32_t pad;
};

// K: uint32_t, or uint64_t for 64-bit keys (NEXT-3); only key equality is used
template <int BLOCK, typename K = uint32_t>
__global__ void __launch_bounds__(BLOCK)
    k_entropy_sorted(const K *__restrict__ keys, uint64_t n, uint64_t chunk,
                     RunPieces *__restrict__ pieces, double *__restrict__ chunk_S, double *__restrict__ out_H,
                     uint32_t *__restrict__ done)
{
    pdl_begin();
    constexpr int NW = BLOCK / 32;
    __shared__ uint32_t s_last;
    __shared__ double s_d[NW];
    __shared__ RunPieces s_wp[NW];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // warp w of the CTA owns the contiguous sub-chunk [c0, c1) of the CTA's chunk
    // (wchunk keys, a multiple of 16): its carry between steps is a warp scan, no
    // block barrier; the warps' boundary pieces are stitched into the CTA's below
    const uint64_t wchunk = chunk / NW;
    const uint64_t c0 = min(n, (uint64_t)blockIdx.x * chunk + warp * wchunk);
    const uint64_t c1 = min(n, c0 + wchunk);
    RunPieces rp{0ull, 0ull, 0u, 0u};
    // a run that began before the sub-chunk enters it unless key[c0] starts a new run
    const bool virt = c0 > 0 && c0 < c1 && keys[c0] == keys[c0 - 1];

    // positions below are sub-chunk-local (32-bit: chunk < 2^32)
    const uint32_t len = (uint32_t)(c1 - c0);
    uint32_t carry = 0;  // local start of the run in progress (0 also when it entered the sub-chunk)
    double S = 0.0;
    const bool vec = ((uintptr_t)keys & 15u) == 0;  // sub-chunk and step starts are multiples of 16 keys
    constexpr uint32_t STEP = 32u * kEntItems;
    const K *kc = keys + c0;
    // keys of the step at t0 for this lane, plus the warp's edge neighbours (lane 0:
    // the key before its first, lane 31: the key after its last; keys past the
    // sub-chunk, up to n, are read too: a run end looks one key ahead)
    auto load = [&](uint32_t t0, K (&k)[kEntItems], K &edge) {
        const uint32_t i0 = t0 + lane * kEntItems;
        if (vec && c0 + i0 + kEntItems <= n) {
            const uint4 *p4 = reinterpret_cast<const uint4 *>(kc + i0);
            if constexpr (sizeof(K) == 4) {
#pragma unroll
                for (int q = 0; q < kEntItems / 4; q++) {
                    const uint4 x = ld_nc_v4(p4 + q);
                    k[4 * q] = x.x;
                    k[4 * q + 1] = x.y;
                    k[4 * q + 2] = x.z;
                    k[4 * q + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < kEntItems / 2; q++) {
                    const uint4 x = ld_nc_v4(p4 + q);
                    k[2 * q] = ((uint64_t)x.y << 32) | x.x;
                    k[2 * q + 1] = ((uint64_t)x.w << 32) | x.z;
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < kEntItems; q++) k[q] = (c0 + i0 + q < n) ? kc[i0 + q] : K(0);
        }
        edge = K(0);
        if (lane == 0 && c0 + i0 > 0 && i0 < len) edge = kc[(int64_t)i0 - 1];
        if (lane == 31 && c0 + i0 + kEntItems < n) edge = kc[i0 + kEntItems];
    };
    const bool last_chunk = c1 == n;
    K k[kEntItems], kn[kEntItems], edge = K(0), edge_n = K(0);
    if (len > 0) load(0, kn, edge_n);
    for (uint32_t t0 = 0; t0 < len; t0 += STEP) {  // warp-uniform trip count
        const uint32_t i0 = t0 + lane * kEntItems;
#pragma unroll
        for (int q = 0; q < kEntItems; q++) k[q] = kn[q];
        edge = edge_n;
        if (t0 + STEP < len) load(t0 + STEP, kn, edge_n);  // next step in flight while this one is scanned
        // neighbours: the previous / next lane's keys; the loaded edges at warp edges
        K prev = __shfl_up_sync(kFull, k[kEntItems - 1], 1);
        K next = __shfl_down_sync(kFull, k[0], 1);
        if (lane == 0) prev = edge;
        if (lane == 31) next = edge;
        // bit q: key q equals its predecessor; starts = the other valid keys
        uint32_t eqm = 0;
#pragma unroll
        for (int q = 0; q < kEntItems; q++) eqm |= (uint32_t)(k[q] == (q ? k[q - 1] : prev)) << q;
        const uint32_t valid = i0 >= len ? 0u : (len - i0 >= (uint32_t)kEntItems ? 0xffffu : (1u << (len - i0)) - 1u);
        const uint32_t stm = ~eqm & valid;
        const uint32_t mine = stm ? i0 + 31u - (uint32_t)__clz(stm) : 0u;  // last local start (0: none; neutral)
        // exclusive max-scan over the warp (lane order = key order), seeded with the carry
        uint32_t incl = max(mine, carry);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(kFull, incl, o);
            if (lane >= (uint32_t)o) incl = max(incl, x);
        }
        const uint32_t up = __shfl_up_sync(kFull, incl, 1);
        uint32_t cur = lane ? up : carry;
        // fast paths (no contribution, no boundary piece): every run of my keys is a single key
        // that ends here, or all my keys sit inside one run that goes on past them; keys at the
        // sub-chunk's edges and partial steps take the loop
        const bool inner = valid == 0xffffu && i0 != 0u && i0 + kEntItems < len;
        const bool singles = inner && eqm == 0u && next != k[kEntItems - 1];
        const bool interior = inner && eqm == 0xffffu && next == k[kEntItems - 1];
        if (!singles && !interior)
#pragma unroll
        for (int q = 0; q < kEntItems; q++) {
            const uint32_t i = i0 + q;
            if (i < len) {
                const bool st = k[q] != (q ? k[q - 1] : prev) || (c0 + i == 0);
                if (st) cur = i;
                const bool end = (last_chunk && i + 1 == len) ||
                                 (q + 1 < kEntItems ? k[q + 1] != k[q] : next != k[q]);
                const bool entered = virt && cur == 0 && !st;  // the run that entered the sub-chunk
                if (end) {
                    if (entered) {
                        rp.pre = i + 1;
                        rp.pre_ends = 1u;
                    } else if (i > cur) {  // runs of one key contribute 1 log2 1 = 0
                        const double c = (double)(i - cur + 1);
                        S += c * log2(c);
                    }
                } else if (i + 1 == len) {  // the last run continues into the next sub-chunk
                    if (entered) rp.pre = len;  // ... and entered it: it crosses the whole sub-chunk
                    else rp.suf = len - cur;
                }
            }
        }
        carry = __shfl_sync(kFull, incl, 31);
    }
    // the warp's pieces: each is set by at most one lane (the one holding that key)
    {
        const uint64_t pre = __reduce_max_sync(kFull, (uint32_t)rp.pre);
        const uint64_t suf = __reduce_max_sync(kFull, (uint32_t)rp.suf);
        const uint32_t pe = __reduce_or_sync(kFull, rp.pre_ends);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S += __shfl_down_sync(kFull, S, o);  // fixed order
        if (lane == 0) {
            s_wp[warp] = RunPieces{pre, suf, pe, 0u};
            s_d[warp] = S;
        }
    }
    __syncthreads();
    // the CTA's pieces from its warps' (fixed order): runs crossing warp boundaries
    // inside the chunk end in a later warp (c log2 c) or continue past the chunk (suf);
    // the run entering the chunk runs through warps while they are crossed whole
    if (threadIdx.x == 0) {
        double t = 0.0;
        RunPieces cp{0ull, 0ull, 0u, 0u};
        for (int w = 0; w < NW; w++) t += s_d[w];
        for (int w = 0; w < NW; w++) {
            uint64_t run = s_wp[w].suf;
            if (run == 0) continue;
            bool ended = false;
            for (int e = w + 1; e < NW; e++) {
                run += s_wp[e].pre;
                if (s_wp[e].pre_ends) {
                    ended = true;
                    break;
                }
            }
            if (ended) t += (double)run * log2((double)run);
            else cp.suf = run;
        }
        if (s_wp[0].pre > 0) {
            uint64_t run = 0;
            for (int e = 0; e < NW; e++) {
                run += s_wp[e].pre;
                if (s_wp[e].pre_ends) {
                    cp.pre_ends = 1u;
                    break;
                }
            }
            cp.pre = run;
        }
        chunk_S[blockIdx.x] = t;
        pieces[blockIdx.x] = cp;
        __threadfence();
        s_last = atomicAdd(done, 1u) == gridDim.x - 1u;  // *done is zeroed before the launch
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // ---- the last CTA to finish: the runs crossing chunk boundaries, then a fixed
    // tree over the chunk sums (the same for whichever CTA is last).  A crossing run has exactly one origin chunk (suf > 0, where
    // it starts); the thread of that chunk follows it forward through chunks it
    // crosses whole (pre > 0, !pre_ends) to the one it ends in.
    {
        __shared__ RunPieces s_pieces[kEntMaxGrid];
        for (uint32_t c = threadIdx.x; c < gridDim.x; c += BLOCK) {
            RunPieces rp;
            rp.pre = __ldcg(&pieces[c].pre);
            rp.suf = __ldcg(&pieces[c].suf);
            rp.pre_ends = __ldcg(&pieces[c].pre_ends);
            s_pieces[c] = rp;
        }
        __syncthreads();
        double t = 0.0;
        for (uint32_t c = threadIdx.x; c < gridDim.x; c += BLOCK) {
            t += __ldcg(&chunk_S[c]);
            uint64_t run = s_pieces[c].suf;
            if (run == 0) continue;
            for (uint32_t e = c + 1; e < gridDim.x; e++) {  // the run continues into chunk e
                run += s_pieces[e].pre;
                if (s_pieces[e].pre_ends) break;
            }
            t += (double)run * log2((double)run);  // run >= 2: it spans a boundary
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(kFull, t, o);
        if (lane == 0) s_d[warp] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < BLOCK / 32; w++) tot += s_d[w];
            const double dn = (double)n;
            const double H = log2(dn) - tot / dn;
            *out_H = H < 0.0 ? 0.0 : H;
        }
    }
}

}  // namespace ahs
