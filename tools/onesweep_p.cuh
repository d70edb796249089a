// onesweep_p.cuh — K6p: the onesweep digit pass of onesweep.cuh (one stable
// 8-bit LSD digit pass, §III.G, Eq. 4) with
// the decoupled look-back taken off the critical path of the tile work.
//
// Warp-specialised persistent CTAs (two per SM): NW worker warps and LBW
// look-back warps.  The workers count, rank and scatter tile t while the
// look-back warps walk the predecessor statuses of tile t-1; the workers
// write tile t-1 out only after ranking tile t:
//
//   workers   | wait keys(t) | count(t) | totals: AGG(t), scan | offsets,
//             |   wait LB(t-1), write-out(t-1) | ticket + TMA(t+1) into the
//             |   freed buffer | rank + scatter(t) |  -> next tile
//   look-back |           ... walk(t-1), INCL(t-1), gofs(t-1) | wait AGG(t)
//             |   walk(t) ...
//
// so a tile's look-back (two L2 round trips under the pass's own streaming
// load, ~40 % of a tile in K6) overlaps the next tile's counting and
// ranking, and the next tile's TMA load overlaps the ranking.  Two tile
// buffers: {ranked, waiting for its look-back} and {being counted/ranked, or
// loading}.  Handoffs use mbarriers (workers -> look-back: totals and digit
// starts ready; look-back -> workers: global offsets ready) and the workers
// synchronise among themselves with a named barrier, so the look-back warps
// never wait on the tile work and vice versa.
//
// Per tile, the work is K6's (onesweep.cuh): early per-warp digit counts
// (shared atomics), tile totals published as AGG statuses before any
// ranking, ranking by ordered shared atomics (one atomic with return per key;
// the host selects this kernel only after the lane-order self-test), scatter
// into an XOR-swizzled reorder buffer, coalesced write-out with the output
// transform fused.  Look-back lanes own DPL consecutive digits each and read
// a predecessor's DPL statuses with one vector load (a warp reads whole
// 1 KiB status rows, coalesced), W predecessors per round.
#pragma once

#include "../paper_2506_20677_b200/csrc/onesweep.cuh"

namespace ahs {

template <int DPL>
struct LbVec;
template <>
struct LbVec<4> {
    using T = uint4;
    static __device__ __forceinline__ T ld(const uint32_t *p)
    {
        T r;
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(p)
                     : "memory");
        return r;
    }
    static __device__ __forceinline__ void st(uint32_t *p, const uint32_t (&v)[4])
    {
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v[0]), "r"(v[1]),
                     "r"(v[2]), "r"(v[3])
                     : "memory");
    }
    static __device__ __forceinline__ uint32_t get(const T &t, int k)
    {
        return k == 0 ? t.x : k == 1 ? t.y : k == 2 ? t.z : t.w;
    }
    static __device__ __forceinline__ T incl0() { return make_uint4(kFlagIncl, kFlagIncl, kFlagIncl, kFlagIncl); }
};
template <>
struct LbVec<2> {
    using T = uint2;
    static __device__ __forceinline__ T ld(const uint32_t *p)
    {
        T r;
        asm volatile("ld.relaxed.gpu.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
        return r;
    }
    static __device__ __forceinline__ void st(uint32_t *p, const uint32_t (&v)[2])
    {
        asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v[0]), "r"(v[1]) : "memory");
    }
    static __device__ __forceinline__ uint32_t get(const T &t, int k) { return k == 0 ? t.x : t.y; }
    static __device__ __forceinline__ T incl0() { return make_uint2(kFlagIncl, kFlagIncl); }
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <bool KV, int NW, int ITEMS, int LBW, typename K = uint32_t, typename V = uint32_t>
struct OnesweepP {
    static constexpr int kWorkers = NW * 32;
    static constexpr int kBlock = (NW + LBW) * 32;
    static constexpr int kTile = kWorkers * ITEMS;
    static constexpr int kSeg = 32 * ITEMS;           // keys per worker warp (its digit table)
    static constexpr int kDPL = kBins / (LBW * 32);   // digits per look-back lane
    static_assert(kDPL == 2 || kDPL == 4, "2 or 4 look-back warps");
    static_assert(kWorkers >= kBins, "one worker thread per digit in the tile scans");
    static_assert(kTile < 65536, "tile positions");
    static_assert((kTile * sizeof(K)) % 16 == 0 && (kTile * sizeof(V)) % 16 == 0, "TMA tile size");
    static constexpr size_t kBufK = (size_t)kTile * sizeof(K);
    static constexpr size_t kBufV = (size_t)kTile * sizeof(V);
    static constexpr size_t kOffK = 0;                                   // keys   [2][TILE]
    static constexpr size_t kOffV = kOffK + 2 * kBufK;                   // values [2][TILE]
    static constexpr size_t kOffCnt = kOffV + (KV ? 2 * kBufV : 0);      // digit tables [NW][256]
    static constexpr size_t kOffAux = kOffCnt + (size_t)NW * kBins * 4;
    // aux: start[2][256], total[2][256], gofs[2][256], wsum[8]
    static constexpr size_t kSmem = kOffAux + (size_t)(6 * kBins + 8) * 4;
};

template <bool KV, int NW, int ITEMS, int LBW, int W = 8, typename K = uint32_t, typename V = uint32_t>
__global__ void __launch_bounds__((NW + LBW) * 32, 2) k_onesweep_p(const PassArgsT<K, V> a)
{
    using C = OnesweepP<KV, NW, ITEMS, LBW, K, V>;
    constexpr int TILE = C::kTile, SEG = C::kSeg, WORKERS = C::kWorkers, DPL = C::kDPL;
    using LV = LbVec<DPL>;
    pdl_begin();
    for (uint32_t i = blockIdx.x * C::kBlock + threadIdx.x; i < a.clear_words; i += gridDim.x * C::kBlock)
        a.status_clear[i] = 0u;
    uint32_t e = a.pass, m = a.npasses;
    if (a.plan) {
        const uint32_t w = a.plan[a.pass];
        if (w == kPassSkip) return;
        e = w >> 8;
        m = w & 255u;
    }
    const bool first = e == 0, last = e + 1 == m;
    const bool to_out = ((m - 1 - e) & 1u) == 0;
    const bool from_out = !first && !to_out;
    const K *__restrict__ keys_in = first ? a.keys_in : (from_out ? a.keys_out : a.keys_tmp);
    const V *__restrict__ vals_in = first ? a.vals_in : (from_out ? a.vals_out : a.vals_tmp);
    K *__restrict__ keys_out = to_out ? a.keys_out : a.keys_tmp;
    V *__restrict__ vals_out = to_out ? a.vals_out : a.vals_tmp;
    const uint32_t n = a.n, shift = a.shift;
    const K in_flip = first ? a.flip : K(0), in_sub = first ? a.sub : K(0);
    const K out_flip = last ? a.flip : K(0), out_add = last ? a.sub : K(0);
    const uint32_t *__restrict__ bucket_base = a.bucket_base;
    uint32_t *__restrict__ status = a.status;
    uint32_t *__restrict__ tile_ticket = a.ticket;
    const uint32_t tma_ok = (((uintptr_t)keys_in & 15u) == 0) && (!KV || ((uintptr_t)vals_in & 15u) == 0);

    extern __shared__ __align__(128) uint8_t smem[];
    K *s_kb = reinterpret_cast<K *>(smem + C::kOffK);
    V *s_vb = reinterpret_cast<V *>(smem + C::kOffV);
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(smem + C::kOffCnt);
    uint32_t *s_start = reinterpret_cast<uint32_t *>(smem + C::kOffAux);  // [2][256]
    uint32_t *s_total = s_start + 2 * kBins;                              // [2][256]
    uint32_t *s_gofs = s_total + 2 * kBins;                               // [2][256]
    uint32_t *s_wsum = s_gofs + 2 * kBins;                                // [8]
    __shared__ __align__(8) uint64_t s_full[2], s_lbready[2], s_lbdone[2];
    __shared__ uint32_t s_ticket[2];
    __shared__ uint32_t s_skew;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t ntiles = (n + TILE - 1) / TILE;
    auto tile_full = [&](uint32_t t) { return (uint64_t)(t + 1) * TILE <= n; };
    auto issue = [&](uint32_t t, uint32_t b) {  // one thread: next tile into buffer b (0 bytes: none / manual)
        const bool tma = t < ntiles && tma_ok && tile_full(t);
        const uint32_t kbytes = (uint32_t)(TILE * sizeof(K)), vbytes = (uint32_t)(TILE * sizeof(V));
        mbar_expect_tx(&s_full[b], tma ? kbytes + (KV ? vbytes : 0u) : 0u);
        if (tma) {
            tma_load_1d(s_kb + b * TILE, keys_in + (size_t)t * TILE, kbytes, &s_full[b]);
            if constexpr (KV) tma_load_1d(s_vb + b * TILE, vals_in + (size_t)t * TILE, vbytes, &s_full[b]);
        }
    };

    if (tid == 0) {
        s_skew = 0u;
        for (int b = 0; b < 2; b++) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_lbready[b], 1);
            mbar_init(&s_lbdone[b], LBW * 32);
        }
        mbar_fence_init();
    }
    for (int i = tid; i < NW * kBins / 4; i += C::kBlock)
        reinterpret_cast<uint4 *>(s_cnt)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    // skewed digit distribution (a digit holds > 1/16 of the keys): warp-uniform fast path
    if (tid < kBins) {
        const uint32_t hi = tid == kBins - 1 ? n : __ldg(&bucket_base[tid + 1]);
        if (hi - __ldg(&bucket_base[tid]) > n / 16u) s_skew = 1u;
    }
    if (tid == 0) {
        const uint32_t t0 = atomicAdd(tile_ticket, 1u);
        s_ticket[0] = t0;
        issue(t0, 0);
    }
    __syncthreads();

    // ================================================================ look-back warps
    if (warp >= (uint32_t)NW) {
        const uint32_t d0 = (tid - WORKERS) * DPL;
        uint32_t base[DPL];
#pragma unroll
        for (int k = 0; k < DPL; k++) base[k] = __ldg(&bucket_base[d0 + k]);
        for (uint32_t j = 0;; j++) {
            const uint32_t bb = j & 1u;
            mbar_wait(&s_lbready[bb], (j >> 1) & 1u);
            const uint32_t tile = s_ticket[bb];
            if (tile >= ntiles) break;
            uint32_t excl[DPL];
#pragma unroll
            for (int k = 0; k < DPL; k++) excl[k] = 0u;
            if (tile > 0) {
                uint32_t need = (1u << DPL) - 1u;  // digits still without an inclusive predecessor
                int jt = (int)tile - 1;
                uint32_t spins = 0;
                while (true) {
                    typename LV::T st[W];
                    const uint32_t *ps = status + (size_t)jt * kBins + d0;
                    if (jt >= W - 1) {
#pragma unroll
                        for (int q = 0; q < W; q++) st[q] = LV::ld(ps - q * kBins);
                    } else {
#pragma unroll
                        for (int q = 0; q < W; q++) st[q] = (jt - q >= 0) ? LV::ld(ps - q * kBins) : LV::incl0();
                    }
                    int used = 0;
                    bool stop = false;
#pragma unroll
                    for (int q = 0; q < W; q++) {
                        if (!stop) {
                            bool pub = true;
#pragma unroll
                            for (int k = 0; k < DPL; k++)
                                pub &= !((need >> k) & 1u) || (LV::get(st[q], k) & ~kCountMask) != 0u;
                            if (!pub) {
                                stop = true;
                            } else {
#pragma unroll
                                for (int k = 0; k < DPL; k++) {
                                    const uint32_t s = LV::get(st[q], k);
                                    if ((need >> k) & 1u) {
                                        excl[k] += s & kCountMask;
                                        if ((s & ~kCountMask) == kFlagIncl) need &= ~(1u << k);
                                    }
                                }
                                used++;
                                if (!need) stop = true;
                            }
                        }
                    }
                    if (!need) break;
                    jt -= used;
                    if (used == 0) {
                        if (++spins > (1u << 26)) __trap();
                        __nanosleep(64);
                    }
                }
                uint32_t incl[DPL];
#pragma unroll
                for (int k = 0; k < DPL; k++) incl[k] = kFlagIncl | (excl[k] + s_total[bb * kBins + d0 + k]);
                LV::st(status + (size_t)tile * kBins + d0, incl);
            }
#pragma unroll
            for (int k = 0; k < DPL; k++) s_gofs[bb * kBins + d0 + k] = base[k] + excl[k] - s_start[bb * kBins + d0 + k];
            mbar_arrive(&s_lbdone[bb]);
        }
        return;
    }

    // ================================================================ worker warps
    auto wbar = [] { asm volatile("bar.sync 1, %0;" ::"n"(WORKERS) : "memory"); };
    const bool skew = s_skew != 0u;
    const uint32_t ltj = lanemask_lt();
    uint32_t *cw = s_cnt + warp * kBins;
    const uint32_t sbase = warp * SEG + lane;

    auto write_out = [&](uint32_t pb, uint32_t pn) {
        const K *sk = s_kb + pb * TILE;
        const V *sv = s_vb + pb * TILE;
        const uint32_t *gofs = s_gofs + pb * kBins;
        if (pn == (uint32_t)TILE) {
#pragma unroll 4
            for (int i = tid; i < TILE; i += WORKERS) {
                const K x = sk[swz(i)];
                const uint32_t o = gofs[digit8(x, shift)] + i;
                keys_out[o] = (x + out_add) ^ out_flip;
                if constexpr (KV) vals_out[o] = sv[swz(i)];
            }
        } else {
            for (uint32_t i = tid; i < pn; i += WORKERS) {
                const K x = sk[swz(i)];
                const uint32_t o = gofs[digit8(x, shift)] + i;
                keys_out[o] = (x + out_add) ^ out_flip;
                if constexpr (KV) vals_out[o] = sv[swz(i)];
            }
        }
    };

    uint32_t prev_n = 0;  // keys of the ranked tile waiting for its look-back (0: none)
    uint32_t it = 0;
    for (;; it++) {
        const uint32_t b = it & 1u;
        mbar_wait(&s_full[b], (it >> 1) & 1u);
        const uint32_t tile = s_ticket[b];
        if (tile >= ntiles) {
            if (tid == 0) mbar_arrive(&s_lbready[b]);  // look-back warps: no more tiles
            break;
        }
        const uint32_t tile_base = tile * (uint32_t)TILE;
        const uint32_t tile_n = min((uint32_t)TILE, n - tile_base);
        K *sk = s_kb + b * TILE;
        V *sv = s_vb + b * TILE;
        if (!(tma_ok && tile_n == (uint32_t)TILE)) {
            for (uint32_t i = tid; i < tile_n; i += WORKERS) {
                sk[i] = ld_nc(keys_in + tile_base + i);
                if constexpr (KV) sv[i] = ld_nc(vals_in + tile_base + i);
            }
            wbar();
        }

        auto tile_work = [&](auto full_c) {
            constexpr bool FULL = decltype(full_c)::value;
            bool wskew = skew;
            // ------------------------------------------------ early counts
            K v[ITEMS];
            [[maybe_unused]] V pv[KV ? ITEMS : 1];
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                const uint32_t idx = sbase + i * 32;
                const bool valid = FULL || idx < tile_n;
                v[i] = ((valid ? sk[idx] : K(0)) ^ in_flip) - in_sub;
                if constexpr (KV) pv[i] = valid ? sv[idx] : V(0);
                const uint32_t d = digit8(v[i], shift);
                if (i == 0 && !wskew) wskew = __all_sync(kFull, d == __shfl_sync(kFull, d, 0));
                if (wskew) {
                    const uint32_t d0 = __shfl_sync(kFull, d, 0);
                    if (__all_sync(kFull, !valid || d == d0)) {
                        const uint32_t vm = FULL ? kFull : __ballot_sync(kFull, valid);
                        if (lane == 0) cw[d0] += __popc(vm);
                        __syncwarp();
                        continue;
                    }
                }
                if (valid) atomicAdd(&cw[d], 1u);
            }
            wbar();

            // ------------------ tile totals: publish AGG, scan -> digit starts
            if (tid < kBins) {
                const uint32_t d = tid;
                uint32_t total = 0;
#pragma unroll
                for (int s = 0; s < NW; s++) total += s_cnt[s * kBins + d];
                st_relaxed(&status[(size_t)tile * kBins + d], (tile == 0 ? kFlagIncl : kFlagAgg) | total);
                s_total[b * kBins + d] = total;
                uint32_t incl = total;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= (uint32_t)o) incl += t;
                }
                if (lane == 31) s_wsum[warp] = incl;
                asm volatile("bar.sync 2, %0;" ::"n"(kBins) : "memory");
                uint32_t before = 0;
#pragma unroll
                for (int w = 0; w < kBins / 32; w++)
                    if (w < (int)warp) before += s_wsum[w];
                s_start[b * kBins + d] = before + incl - total;
            }
            wbar();
            if (tid == 0) mbar_arrive(&s_lbready[b]);  // totals and starts of this tile: look-back may run
            // per-warp digit offsets in the tile (digit start + earlier warps' counts)
            if (tid < kBins) {
                uint32_t run = s_start[b * kBins + tid];
#pragma unroll
                for (int s = 0; s < NW; s++) {
                    uint32_t *p = &s_cnt[s * kBins + tid];
                    const uint32_t c = *p;
                    *p = run;
                    run += c;
                }
            }
            // ------------------------- write out the previous (ranked) tile
            if (prev_n) {
                mbar_wait(&s_lbdone[b ^ 1u], ((it - 1) >> 1) & 1u);
                write_out(b ^ 1u, prev_n);
            }
            wbar();
            // the previous tile's buffer is free: next ticket, its keys by TMA
            if (tid == 0) {
                const uint32_t nt = atomicAdd(tile_ticket, 1u);
                s_ticket[b ^ 1u] = nt;
                fence_proxy_async();
                issue(nt, b ^ 1u);
            }
            // ---------------------------------- rank + scatter in digit order
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                const uint32_t idx = sbase + i * 32;
                const bool valid = FULL || idx < tile_n;
                const uint32_t dd = digit8(v[i], shift);
                uint32_t pos = 0;
                bool done = false;
                if (wskew) {
                    const uint32_t d0 = __shfl_sync(kFull, dd, 0);
                    if (__all_sync(kFull, !valid || dd == d0)) {
                        const uint32_t vm = FULL ? kFull : __ballot_sync(kFull, valid);
                        const uint32_t c = cw[d0];
                        pos = c + __popc(vm & ltj);
                        __syncwarp();
                        if (lane == 0) cw[d0] = c + __popc(vm);
                        done = true;
                    }
                }
                if (!done && valid) pos = atomicAdd(&cw[dd], 1u);  // lanes served in lane order (self-tested)
                if (valid) {
                    sk[swz(pos)] = v[i];
                    if constexpr (KV) sv[swz(pos)] = pv[i];
                }
                __syncwarp();
            }
            // this warp's digit table: cleared for the next tile
            {
                uint4 *t4 = reinterpret_cast<uint4 *>(cw);
#pragma unroll
                for (int q = 0; q < kBins / 4 / 32; q++) t4[q * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
            }
        };
        if (tile_n == (uint32_t)TILE) tile_work(std::true_type{});
        else tile_work(std::false_type{});
        prev_n = tile_n;
    }
    // the last ranked tile
    if (prev_n) {
        const uint32_t pb = (it - 1) & 1u;
        mbar_wait(&s_lbdone[pb], ((it - 1) >> 1) & 1u);
        wbar();  // every worker's scatter into pb is complete
        write_out(pb, prev_n);
    }
}

}  // namespace ahs
