// onesweep_b.cuh — K6b: the onesweep digit pass of onesweep.cuh (one stable
// 8-bit LSD digit pass, §III.G, Eq. 4) with
// the write-out done by TMA bulk stores, one per digit run.
//
// K6 writes a ranked tile out with one scalar global store per key (plus a
// shared load of the key and of its digit's offset).  Here the decoupled
// look-back runs before the ranking, so each digit's global destination g0 is
// known when the keys are scattered into shared memory; digit d's run is
// placed at a shared slot ps[d] with ps[d] = g0[d] (mod 4) (at most 3 slots of
// padding per digit: ps[d] in [start[d] + 3d, start[d] + 3d + 3]), so the
// 16-byte-aligned body of every run is one cp.async.bulk shared -> global
// copy issued by the digit's thread; the <= 3 keys before and after the body
// are plain stores.  The output transform is applied in the scatter.  The
// reorder buffer is then not swizzled (a bulk copy reads contiguous slots).
//
// A tile buffer is refilled (TMA load of the tile after next) only after the
// bulk copies that read it have finished reading (cp.async.bulk.wait_group.read
// before the barrier that precedes the refill).  Ordered ranking only (the
// lane-order self-test of onesweep.cuh), 32-bit keys and values.
#pragma once

#include "../paper_2506_20677_b200/csrc/onesweep.cuh"

namespace ahs {

__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <bool KV, int BLOCK, int ITEMS>
struct OnesweepB {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * ITEMS;
    static constexpr int kTileP = kTile + 3 * kBins + 4;  // + alignment padding of the digit runs
    static constexpr int kTPD = BLOCK / kBins;
    static_assert(kTile % 4 == 0 && kTileP % 4 == 0, "16-byte buffers");
    static constexpr size_t kOffK = 0;                                  // keys   [2][TILEP]
    static constexpr size_t kOffV = kOffK + 2 * (size_t)kTileP * 4;     // values [2][TILEP]
    static constexpr size_t kOffCnt = kOffV + (KV ? 2 * (size_t)kTileP * 4 : 0);
    static constexpr size_t kOffAux = kOffCnt + (size_t)kWarps * kBins * 4;
    // aux: part[2][256], start[256], ps[256], g0[256], tot[256], wsum[8]
    static constexpr size_t kSmem = kOffAux + (size_t)(6 * kBins + 8) * 4;
};

template <bool KV, int BLOCK, int ITEMS, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep_b(const PassArgs a)
{
    using K = uint32_t;
    using V = uint32_t;
    pdl_begin();
    auto clear_other = [&] {
        if (a.plan && a.plan[a.pass + 1] == kPassSkip) return;
        for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < a.clear_words; i += gridDim.x * BLOCK)
            a.status_clear[i] = 0u;
    };
    uint32_t e = a.pass, m = a.npasses, shift = a.shift;
    if (a.plan) {
        const uint32_t w = a.plan[a.pass];
        if (w == kPassSkip) {
            clear_other();
            return;
        }
        e = (w >> 8) & 255u;
        m = w & 255u;
        shift = w >> 16;
    }
    const bool first = e == 0, last = e + 1 == m;
    const bool to_out = ((m - 1 - e) & 1u) == 0;
    const bool from_out = !first && !to_out;
    const K *__restrict__ keys_in = first ? a.keys_in : (from_out ? a.keys_out : a.keys_tmp);
    const V *__restrict__ vals_in = first ? a.vals_in : (from_out ? a.vals_out : a.vals_tmp);
    K *__restrict__ keys_out = to_out ? a.keys_out : a.keys_tmp;
    V *__restrict__ vals_out = to_out ? a.vals_out : a.vals_tmp;
    const uint32_t n = a.n;
    const K in_flip = first ? a.flip : K(0), in_sub = first ? a.sub : K(0);
    const K out_flip = last ? a.flip : K(0), out_add = last ? a.sub : K(0);
    const uint32_t *__restrict__ bucket_base = a.bucket_base;
    uint32_t *__restrict__ status = a.status;
    uint32_t *__restrict__ tile_ticket = a.ticket;
    const uint32_t tma_ok = (((uintptr_t)keys_in & 15u) == 0) && (!KV || ((uintptr_t)vals_in & 15u) == 0);
    const bool wb_ok = (((uintptr_t)keys_out & 15u) == 0) && (!KV || ((uintptr_t)vals_out & 15u) == 0);

    using C = OnesweepB<KV, BLOCK, ITEMS>;
    constexpr int TILE = C::kTile, TILEP = C::kTileP, SEG = 32 * ITEMS;
    extern __shared__ __align__(128) uint8_t smem[];
    K *s_kb = reinterpret_cast<K *>(smem + C::kOffK);
    V *s_vb = reinterpret_cast<V *>(smem + C::kOffV);
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(smem + C::kOffCnt);
    uint32_t *s_part = reinterpret_cast<uint32_t *>(smem + C::kOffAux);
    uint32_t *s_start = s_part + 2 * kBins;
    uint32_t *s_ps = s_start + kBins;
    uint32_t *s_g0 = s_ps + kBins;
    uint32_t *s_tot = s_g0 + kBins;
    uint32_t *s_wsum = s_tot + kBins;
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_ticket[2];

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t ntiles = (n + TILE - 1) / TILE;
    const uint32_t ltj = lanemask_lt();

    auto tile_full = [&](uint32_t t) { return (uint64_t)(t + 1) * TILE <= n; };
    auto issue = [&](uint32_t t, uint32_t b) {
        const uint32_t bytes = (uint32_t)(TILE * 4);
        mbar_expect_tx(&s_bar[b], bytes * (KV ? 2u : 1u));
        tma_load_1d(s_kb + b * TILEP, keys_in + (size_t)t * TILE, bytes, &s_bar[b]);
        if constexpr (KV) tma_load_1d(s_vb + b * TILEP, vals_in + (size_t)t * TILE, bytes, &s_bar[b]);
    };

    __shared__ uint32_t s_skew;
    if (tid == 0) s_skew = 0u;
    __syncthreads();
    if (tid < kBins) {
        const uint32_t hi = tid == kBins - 1 ? n : __ldg(&bucket_base[tid + 1]);
        if (hi - __ldg(&bucket_base[tid]) > n / 16u) s_skew = 1u;
    }
    for (int i = tid; i < C::kWarps * kBins / 4; i += BLOCK)
        reinterpret_cast<uint4 *>(s_cnt)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_fence_init();
        const uint32_t t0 = atomicAdd(tile_ticket, 1u);
        s_ticket[0] = t0;
        if (t0 < ntiles && tma_ok && tile_full(t0)) issue(t0, 0);
    }
    __syncthreads();

    const bool skew = s_skew != 0u;
    uint32_t phase = 0;
    for (uint32_t iter = 0;; iter++) {
        const uint32_t b = iter & 1u;
        const uint32_t tile = s_ticket[b];
        if (tile >= ntiles) break;
        const uint32_t tile_base = tile * (uint32_t)TILE;
        const uint32_t tile_n = min((uint32_t)TILE, n - tile_base);
        const bool full = tile_n == (uint32_t)TILE;
        K *sk = s_kb + b * TILEP;
        V *sv = s_vb + b * TILEP;
        if (tma_ok && full) {
            mbar_wait(&s_bar[b], (phase >> b) & 1u);
            phase ^= 1u << b;
        } else {
            for (uint32_t i = tid; i < tile_n; i += BLOCK) {
                sk[i] = ld_nc(keys_in + tile_base + i);
                if constexpr (KV) sv[i] = ld_nc(vals_in + tile_base + i);
            }
            __syncthreads();
        }

        auto tile_work = [&](auto full_c) {
            constexpr bool FULL = decltype(full_c)::value;
            bool wskew = skew;
            K v[ITEMS];
            [[maybe_unused]] V pv[KV ? ITEMS : 1];
            uint32_t *cw = s_cnt + warp * kBins;
            const uint32_t sbase = warp * SEG + lane;
#pragma unroll
            for (int it = 0; it < ITEMS; it++) {
                const uint32_t idx = sbase + it * 32;
                const bool valid = FULL || idx < tile_n;
                v[it] = ((valid ? sk[idx] : K(0)) ^ in_flip) - in_sub;
                if constexpr (KV) pv[it] = valid ? sv[idx] : V(0);
                const uint32_t d = digit8(v[it], shift);
                if (it == 0 && !wskew) wskew = __all_sync(kFull, d == __shfl_sync(kFull, d, 0));
                if (valid) atomicAdd(&cw[d], 1u);
            }
            // the bulk copies of the previous tile (other buffer) have read their source
            // before the barrier that precedes the refill of that buffer
            bulk_wait_read();
            __syncthreads();

            // ------------------ per-digit totals, publish aggregate, tile scan, look-back
            const uint32_t d = tid & (kBins - 1), part = tid / kBins;
            constexpr int SPP = C::kWarps / C::kTPD;
            uint32_t psum = 0;
            if (C::kTPD == 2 || tid < kBins) {
#pragma unroll 8
                for (int s = 0; s < SPP; s++) psum += s_cnt[(part * SPP + s) * kBins + d];
            }
            if constexpr (C::kTPD == 2) {
                s_part[part * kBins + d] = psum;
                __syncthreads();
            }
            if (tid < kBins) {
                const uint32_t total = C::kTPD == 2 ? s_part[d] + s_part[kBins + d] : psum;
                st_relaxed(&status[(size_t)tile * kBins + d], (tile == 0 ? kFlagIncl : kFlagAgg) | total);
                uint32_t incl = total;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= (uint32_t)o) incl += t;
                }
                if (lane == 31) s_wsum[warp] = incl;
                asm volatile("bar.sync 1, %0;" ::"n"(kBins) : "memory");
                uint32_t before = 0;
#pragma unroll
                for (int w = 0; w < kBins / 32; w++)
                    if (w < (int)warp) before += s_wsum[w];
                const uint32_t start = before + incl - total;
                uint32_t excl = 0;
                if (tile > 0) {
                    int jt = (int)tile - 1;
                    uint32_t spins = 0;
                    while (true) {
                        uint32_t st[kLookback];
                        if (jt >= kLookback - 1) {
                            const uint32_t *ps = status + (size_t)jt * kBins + d;
#pragma unroll
                            for (int q = 0; q < kLookback; q++) st[q] = ld_relaxed(ps - q * kBins);
                        } else {
#pragma unroll
                            for (int q = 0; q < kLookback; q++)
                                st[q] = (jt - q >= 0) ? ld_relaxed(&status[(size_t)(jt - q) * kBins + d]) : kFlagIncl;
                        }
                        int used = 0;
                        bool fin = false, stop = false;
#pragma unroll
                        for (int q = 0; q < kLookback; q++) {
                            if (!stop) {
                                const uint32_t flag = st[q] & ~kCountMask;
                                if (flag == 0u) {
                                    stop = true;
                                } else {
                                    excl += st[q] & kCountMask;
                                    used++;
                                    if (flag == kFlagIncl) fin = stop = true;
                                }
                            }
                        }
                        if (fin) break;
                        jt -= used;
                        if (used == 0) {
                            if (++spins > kLookbackSpinLimit) {
                                if (!a.fault) __trap();
                                atomicExch(a.fault, 1u);
                                break;
                            }
                            __nanosleep(64);
                        }
                    }
                    st_relaxed(&status[(size_t)tile * kBins + d], kFlagIncl | (excl + total));
                }
                const uint32_t g0 = __ldg(&bucket_base[d]) + excl;
                const uint32_t lo = start + 3u * d;
                s_ps[d] = lo + ((g0 - lo) & 3u);
                s_g0[d] = g0;
                s_tot[d] = total;
            }
            __syncthreads();
            // next tile: ticket + TMA load into the other buffer (its bulk copies have read it)
            if (tid == 0) {
                const uint32_t nt = atomicAdd(tile_ticket, 1u);
                s_ticket[b ^ 1u] = nt;
                if (nt < ntiles && tma_ok && tile_full(nt)) {
                    fence_proxy_async();
                    issue(nt, b ^ 1u);
                }
            }
            // per-warp digit offsets (run start + earlier warps)
            if (C::kTPD == 2 || tid < kBins) {
                uint32_t run = s_ps[d] + (part ? s_part[d] : 0u);
#pragma unroll 8
                for (int s = 0; s < SPP; s++) {
                    uint32_t *p = &s_cnt[(part * SPP + s) * kBins + d];
                    const uint32_t c = *p;
                    *p = run;
                    run += c;
                }
            }
            __syncthreads();

            // ------------------------------------- rank + scatter (output transform fused)
#pragma unroll
            for (int it = 0; it < ITEMS; it++) {
                const uint32_t idx = sbase + it * 32;
                const bool valid = FULL || idx < tile_n;
                const uint32_t dd = digit8(v[it], shift);
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
                if (!done && valid) pos = atomicAdd(&cw[dd], 1u);
                if (valid) {
                    sk[pos] = (v[it] + out_add) ^ out_flip;
                    if constexpr (KV) sv[pos] = pv[it];
                }
                __syncwarp();
            }
            {
                uint4 *t4 = reinterpret_cast<uint4 *>(s_cnt + warp * kBins);
#pragma unroll
                for (int q = 0; q < kBins / 4 / 32; q++) t4[q * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
            }
            fence_proxy_async();  // the scatter's shared writes before the bulk copies read them
            __syncthreads();

            // ------------------------------------------------------- write out
            if (tid < kBins) {
                const uint32_t cnt = s_tot[d];
                if (cnt) {
                    const uint32_t ps = s_ps[d], g0 = s_g0[d];
                    if (wb_ok) {
                        const uint32_t head = min(cnt, (4u - (g0 & 3u)) & 3u);
                        const uint32_t body = (cnt - head) & ~3u;
                        for (uint32_t i = 0; i < head; i++) {
                            keys_out[g0 + i] = sk[ps + i];
                            if constexpr (KV) vals_out[g0 + i] = sv[ps + i];
                        }
                        if (body) {
                            bulk_store(keys_out + g0 + head, sk + ps + head, body * 4u);
                            if constexpr (KV) bulk_store(vals_out + g0 + head, sv + ps + head, body * 4u);
                            bulk_commit();
                        }
                        for (uint32_t i = head + body; i < cnt; i++) {
                            keys_out[g0 + i] = sk[ps + i];
                            if constexpr (KV) vals_out[g0 + i] = sv[ps + i];
                        }
                    } else {
                        for (uint32_t i = 0; i < cnt; i++) {
                            keys_out[g0 + i] = sk[ps + i];
                            if constexpr (KV) vals_out[g0 + i] = sv[ps + i];
                        }
                    }
                }
            }
        };
        if (full) tile_work(std::true_type{});
        else tile_work(std::false_type{});
        __syncthreads();
    }
    bulk_wait_all();
    clear_other();
}

}  // namespace ahs
