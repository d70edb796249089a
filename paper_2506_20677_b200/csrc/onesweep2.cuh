// onesweep2.cuh — K6 v2: one stable LSD digit pass, onesweep style (PAPER.md
// §III.G: each pass a stable counting sort by one digit; Eq. 4
// line 360), generalised over the digit width and rewritten for fewer shared-
// memory operations on skewed digits.  Same pass chain, statuses, look-back and
// ordered ranking as K6 (onesweep.cuh; the masked fallback stays there).
//
//   BITS        8 (the radix passes), 10 (the single stable scatter of key-value
//               COUNTING with k <= 1024, Listing 2) or 11 (the
//               3 x 11-bit digit-width experiment, NEXT-1).  Above 8 bits the
//               per-warp digit tables hold packed 16-bit counters (a tile has
//               < 2^16 keys), so a 1024-digit table is 2 KiB per warp.
//   variants    the tile loop is instantiated per (input transform, output
//               transform): only the first executed pass of a chain maps key ->
//               (key ^ flip) - min, only the last maps back.  Picked once per
//               launch from the device pass plan (NEXT-1).
//   hot digits  the up to four digits holding more than 1/32 of the pass's keys
//               (read off the pass's digit histogram at launch) are counted and
//               ranked with warp ballots and per-warp running offsets in
//               registers: the lanes of one shared atomic *with return* that
//               hit the same word are served one wavefront each, so a 64 % digit
//               (cfg3's last pass) would cost ~20 wavefronts per 32 keys on the
//               rank atomic alone.  Other digits keep the one-atomic ranking.
//   tile scan   totals, the tile's exclusive scan and the per-warp offsets are
//               one phase of the scan threads (each owns BINS / BLOCK digits, at
//               least one), one named barrier among them.
//
// Per tile: early per-warp counts -> AGG statuses -> scan + offsets -> rank +
// scatter into the XOR-swizzled reorder buffer -> decoupled look-back (INCL)
// -> coalesced write-out with the output transform fused.
#pragma once

#include "onesweep.cuh"

// development ablations (tools/passbench.cu only; wrong results): bit 3 no look-back
#ifndef AHS_OS2_ABL
#define AHS_OS2_ABL 0
#endif

namespace ahs {

// HOTCFG: number of hot digits (bits 0-3, 0 = none), share threshold 2^-t (bits 4-7),
// ballot counting of hot digits in the early counts too (bit 8; otherwise only the rank)
constexpr int hotcfg(int nh, int t, bool count) { return nh | (t << 4) | (count ? 256 : 0); }
constexpr int kHotDefault = hotcfg(1, 3, false);

template <bool KV, int BLOCK, int ITEMS, int BITS = 8, typename K = uint32_t, typename V = uint32_t,
          int HOTCFG = kHotDefault>
struct Onesweep2 {
    static constexpr int kBins = 1 << BITS;
    static constexpr bool kPacked = BITS > 8;                          // 16-bit packed counters
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * ITEMS;
    static constexpr int kSeg = 32 * ITEMS;                            // keys per warp (its table)
    static constexpr int kDPT = kBins >= BLOCK ? kBins / BLOCK : 1;    // digits per scan thread
    static constexpr int kNT = kBins / kDPT;                           // scan threads
    static constexpr int kTabWords = kPacked ? kBins / 2 : kBins;      // words per warp table
    static constexpr int kHot = (HOTCFG & 15) ? (HOTCFG & 15) : 1;     // hot digit slots
    static constexpr bool kHotOn = (HOTCFG & 15) != 0;
    static constexpr int kHotShift = (HOTCFG >> 4) & 15;               // share > 2^-kHotShift
    static constexpr bool kHotCount = (HOTCFG & 256) != 0;
    static_assert(BITS >= 8 && BITS <= 11, "8- to 11-bit digits (9: tools/passbench.cu only)");
    static_assert(BLOCK % 128 == 0 && BLOCK >= 256 && BLOCK <= 512, "256, 384 or 512 threads");
    static_assert(kBins <= BLOCK || kBins % BLOCK == 0, "scan threads own whole digit groups");
    static_assert(!kPacked || kDPT % 2 == 0, "packed tables: a scan thread owns whole words");
    static_assert(kDPT <= 4, "look-back vector width");
    static_assert(kTile < 65536, "16-bit tile positions");
    static_assert((kTile * sizeof(K)) % 16 == 0 && (kTile * sizeof(V)) % 16 == 0, "TMA tile size");
    static constexpr size_t kBufK = (size_t)kTile * sizeof(K);
    static constexpr size_t kBufV = (size_t)kTile * sizeof(V);
    static constexpr size_t kOffK = 0;
    static constexpr size_t kOffV = kOffK + 2 * kBufK;
    static constexpr size_t kOffCnt = kOffV + (KV ? 2 * kBufV : 0);
    static constexpr size_t kOffAux = kOffCnt + (size_t)kWarps * kTabWords * 4;
    // aux: start[BINS], gofs[BINS], wsum[32]
    static constexpr size_t kSmem = kOffAux + (size_t)(2 * kBins + 32) * 4;
};

namespace os2 {
// DPT consecutive look-back statuses of one predecessor tile in one load
template <int DPT>
struct Vec {
    uint32_t w[DPT];
};
template <int DPT>
__device__ __forceinline__ Vec<DPT> ld_status(const uint32_t *p)
{
    Vec<DPT> r;
    if constexpr (DPT == 1) {
        r.w[0] = ld_relaxed(p);
    } else if constexpr (DPT == 2) {
        asm volatile("ld.relaxed.gpu.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.w[0]), "=r"(r.w[1]) : "l"(p) : "memory");
    } else {
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                     : "l"(p)
                     : "memory");
    }
    return r;
}
template <int DPT>
__device__ __forceinline__ void st_status(uint32_t *p, const uint32_t (&v)[DPT])
{
    if constexpr (DPT == 1) {
        st_relaxed(p, v[0]);
    } else if constexpr (DPT == 2) {
        asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v[0]), "r"(v[1]) : "memory");
    } else {
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                     "r"(v[3])
                     : "memory");
    }
}
}  // namespace os2

template <bool KV, int BLOCK, int ITEMS, int BITS, bool TIN, bool TOUT, typename K, typename V, int HOTCFG>
__device__ __forceinline__ void onesweep2_body(const PassArgsT<K, V> &a, const K *__restrict__ keys_in,
                                               const V *__restrict__ vals_in, K *__restrict__ keys_out,
                                               V *__restrict__ vals_out, const uint32_t shift)
{
    using C = Onesweep2<KV, BLOCK, ITEMS, BITS, K, V, HOTCFG>;
    constexpr int TILE = C::kTile, SEG = C::kSeg, NWARP = C::kWarps, BINS = C::kBins, DPT = C::kDPT,
                  NT = C::kNT, TW = C::kTabWords, NHOT = C::kHot;
    constexpr bool PACKED = C::kPacked;
    constexpr uint32_t KB = sizeof(K), VB = sizeof(V);
    const uint32_t n = a.n;
    const K flip = a.flip, subv = a.sub;
    const uint32_t *__restrict__ bucket_base = a.bucket_base;
    uint32_t *__restrict__ status = a.status;
    uint32_t *__restrict__ tile_ticket = a.ticket;
    const uint32_t tma_ok = (((uintptr_t)keys_in & 15u) == 0) && (!KV || ((uintptr_t)vals_in & 15u) == 0);

    extern __shared__ __align__(128) uint8_t smem[];
    K *s_kb = reinterpret_cast<K *>(smem + C::kOffK);
    V *s_vb = reinterpret_cast<V *>(smem + C::kOffV);
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(smem + C::kOffCnt);
    uint32_t *s_start = reinterpret_cast<uint32_t *>(smem + C::kOffAux);
    uint32_t *s_gofs = s_start + BINS;
    uint32_t *s_wsum = s_gofs + BINS;
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_ticket[2];
    __shared__ uint32_t s_hot[NHOT];
    __shared__ unsigned long long s_best[BLOCK / 32];

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t ntiles = (n + TILE - 1) / TILE;
    const uint32_t ltj = lanemask_lt();
    uint32_t *const cw = s_cnt + warp * TW;  // this warp's digit table
    auto digit = [&](K v) -> uint32_t { return (uint32_t)(v >> shift) & (uint32_t)(BINS - 1); };
    // per-warp table: 32-bit counters (8-bit digits) or two 16-bit counters per word
    auto t_inc = [&](uint32_t d) {
        if constexpr (PACKED) atomicAdd(&cw[d >> 1], 1u << ((d & 1u) << 4));
        else atomicAdd(&cw[d], 1u);
    };
    auto t_rank = [&](uint32_t d) -> uint32_t {  // lanes of one instruction served in lane order (self-tested)
        if constexpr (PACKED) return (atomicAdd(&cw[d >> 1], 1u << ((d & 1u) << 4)) >> ((d & 1u) << 4)) & 0xffffu;
        else return atomicAdd(&cw[d], 1u);
    };
    auto t_get = [&](uint32_t d) -> uint32_t {
        if constexpr (PACKED) return (cw[d >> 1] >> ((d & 1u) << 4)) & 0xffffu;
        else return cw[d];
    };
    auto t_add = [&](uint32_t d, uint32_t c) {  // one lane; no other lane touches the entry
        if constexpr (PACKED) cw[d >> 1] += c << ((d & 1u) << 4);
        else cw[d] += c;
    };
    auto tile_full = [&](uint32_t t) { return (uint64_t)(t + 1) * TILE <= n; };
    auto issue = [&](uint32_t t, uint32_t b) {
        const uint32_t kbytes = (uint32_t)(TILE * KB), vbytes = (uint32_t)(TILE * VB);
        mbar_expect_tx(&s_bar[b], kbytes + (KV ? vbytes : 0u));
        tma_load_1d(s_kb + b * TILE, keys_in + (size_t)t * TILE, kbytes, &s_bar[b]);
        if constexpr (KV) tma_load_1d(s_vb + b * TILE, vals_in + (size_t)t * TILE, vbytes, &s_bar[b]);
    };
    auto digit_count = [&](uint32_t d) -> uint32_t {
        const uint32_t hi = d == (uint32_t)BINS - 1 ? n : __ldg(&bucket_base[d + 1]);
        return hi - __ldg(&bucket_base[d]);
    };

    for (int i = tid; i < NWARP * TW / 4; i += BLOCK)
        reinterpret_cast<uint4 *>(s_cnt)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_fence_init();
        const uint32_t t0 = atomicAdd(tile_ticket, 1u);
        s_ticket[0] = t0;
        if (t0 < ntiles && tma_ok && tile_full(t0)) issue(t0, 0);
    }
    // hot digits of this pass: up to NHOT digits with more than n >> kHotShift keys, by block argmax
    for (int k = 0; k < (C::kHotOn ? NHOT : 0); k++) {
        unsigned long long best = 0ull;  // count << 32 | (BINS - 1 - d): ties to the smaller digit
        for (uint32_t d = tid; d < (uint32_t)BINS; d += BLOCK) {
            bool taken = false;
            for (int q = 0; q < k; q++) taken |= s_hot[q] == d;
            const uint32_t c = taken ? 0u : digit_count(d);
            const unsigned long long key = ((unsigned long long)c << 32) | (uint32_t)(BINS - 1 - d);
            if (c > (n >> C::kHotShift) && key > best) best = key;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(kFull, best, o);
            best = x > best ? x : best;
        }
        if (lane == 0) s_best[warp] = best;
        __syncthreads();
        if (tid == 0) {
            unsigned long long m = 0ull;
            for (int w = 0; w < BLOCK / 32; w++) m = s_best[w] > m ? s_best[w] : m;
            s_hot[k] = m ? (uint32_t)(BINS - 1) - (uint32_t)(m & 0xffffffffull) : 0xffffffffu;
        }
        __syncthreads();
    }
    __syncthreads();  // barriers, first ticket, cleared tables and the hot digits are visible
    uint32_t hot[NHOT];
#pragma unroll
    for (int k = 0; k < NHOT; k++) hot[k] = C::kHotOn ? s_hot[k] : 0xffffffffu;
    const bool has_hot = C::kHotOn && hot[0] != 0xffffffffu;
    int nh = 0;  // hot digits in use (the slots are filled in order)
#pragma unroll
    for (int k = 0; k < NHOT; k++) nh += hot[k] != 0xffffffffu;

    // write-out read slots of tid + k * BLOCK for the 512-thread CTA: swz(i) = i ^ ((i >> 5) & 31)
    // with (i >> 5) & 31 = warp + 16 (k & 1)
    const uint32_t wo0 = (tid & ~31u) | (lane ^ warp);
    const uint32_t wo1 = (tid & ~31u) | (lane ^ ((warp + 16u) & 31u));

    uint32_t phase = 0;
    for (uint32_t iter = 0;; iter++) {
        const uint32_t b = iter & 1u;
        const uint32_t tile = s_ticket[b];
        if (tile >= ntiles) break;
        const uint32_t tile_base = tile * (uint32_t)TILE;
        const uint32_t tile_n = min((uint32_t)TILE, n - tile_base);
        const bool full = tile_n == (uint32_t)TILE;
        K *sk = s_kb + b * TILE;
        V *sv = s_vb + b * TILE;
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
            K v[ITEMS];
            [[maybe_unused]] V pv[KV ? ITEMS : 1];
            const uint32_t sbase = warp * SEG + lane;  // slot of item 0
            auto valid_at = [&](int i) { return FULL || sbase + (uint32_t)i * 32u < tile_n; };
            // all loads first (the table atomics may alias the tile buffer for the compiler)
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                const uint32_t idx = sbase + i * 32;
                K x = valid_at(i) ? sk[idx] : K(0);
                if constexpr (TIN) x = (x ^ flip) - subv;
                v[i] = x;
                if constexpr (KV) pv[i] = valid_at(i) ? sv[idx] : V(0);
            }
            // loop form for this warp and tile: the warp-uniform-digit form (this warp's first 32
            // keys share a digit: sorted runs), hot digits (skewed pass), or the plain form
            const uint32_t dl0 = __shfl_sync(kFull, digit(v[0]), 0);  // every lane: no short circuit
            const bool uni0 = __all_sync(kFull, !valid_at(0) || digit(v[0]) == dl0);
            const int form = uni0 ? 1 : has_hot ? 2 : 0;
            // --------------------------------------------- early counts
            if (form == 0) {
#pragma unroll
                for (int i = 0; i < ITEMS; i++)
                    if (valid_at(i)) t_inc(digit(v[i]));
            } else if (form == 1 || !C::kHotCount) {
                // same-address lanes of an atomic without return are merged: plain counts
#pragma unroll
                for (int i = 0; i < ITEMS; i++)
                    if (valid_at(i)) t_inc(digit(v[i]));
            } else {
                uint32_t hc[NHOT];
#pragma unroll
                for (int k = 0; k < NHOT; k++) hc[k] = 0;
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const bool valid = valid_at(i);
                    const uint32_t d = digit(v[i]);
                    bool h = false;
#pragma unroll
                    for (int k = 0; k < NHOT; k++) {
                        const bool mine = valid && d == hot[k];
                        hc[k] += __popc(__ballot_sync(kFull, mine));
                        h |= mine;
                    }
                    if (valid && !h) t_inc(d);
                }
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < NHOT; k++)
                        if (hot[k] != 0xffffffffu && hc[k]) t_add(hot[k], hc[k]);
                }
            }
            __syncthreads();

            // ---------- totals -> AGG statuses, tile scan, per-warp offsets (scan threads)
            const uint32_t d0 = tid * DPT;
            uint32_t tot[DPT];
            if (tid < (uint32_t)NT) {
                uint32_t sum = 0, pre[DPT];
#pragma unroll
                for (int j = 0; j < DPT; j++) tot[j] = 0;
#pragma unroll 4
                for (int w = 0; w < NWARP; w++) {
                    if constexpr (PACKED) {
#pragma unroll
                        for (int j = 0; j < DPT; j += 2) {
                            const uint32_t x = s_cnt[w * TW + (d0 + j) / 2];
                            tot[j] += x & 0xffffu;
                            tot[j + 1] += x >> 16;
                        }
                    } else {
                        tot[0] += s_cnt[w * TW + d0];
                    }
                }
                uint32_t sts[DPT];
#pragma unroll
                for (int j = 0; j < DPT; j++) {
                    pre[j] = sum;
                    sum += tot[j];
                    sts[j] = (tile == 0 ? kFlagIncl : kFlagAgg) | tot[j];
                }
                os2::st_status<DPT>(&status[(size_t)tile * BINS + d0], sts);
                uint32_t incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= (uint32_t)o) incl += t;
                }
                if (lane == 31) s_wsum[warp] = incl;
                asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
                uint32_t before = 0;
#pragma unroll
                for (int w = 0; w < NT / 32; w++)
                    if (w < (int)warp) before += s_wsum[w];
                const uint32_t base = before + incl - sum;
                uint32_t run[DPT];
#pragma unroll
                for (int j = 0; j < DPT; j++) {
                    run[j] = base + pre[j];
                    s_start[d0 + j] = run[j];
                }
                // per-warp offsets: digit start + earlier warps' counts (tile positions < 2^16)
#pragma unroll 4
                for (int w = 0; w < NWARP; w++) {
                    if constexpr (PACKED) {
#pragma unroll
                        for (int j = 0; j < DPT; j += 2) {
                            uint32_t *p = &s_cnt[w * TW + (d0 + j) / 2];
                            const uint32_t x = *p;
                            *p = run[j] | (run[j + 1] << 16);
                            run[j] += x & 0xffffu;
                            run[j + 1] += x >> 16;
                        }
                    } else {
                        uint32_t *p = &s_cnt[w * TW + d0];
                        const uint32_t c = *p;
                        *p = run[0];
                        run[0] += c;
                    }
                }
            }
            __syncthreads();

            // ------------------------------------- rank + scatter in digit order
            auto scatter = [&](uint32_t pos, int i) {
                const uint32_t sp = pos ^ ((pos >> 5) & 31u);
                sk[sp] = v[i];
                if constexpr (KV) sv[sp] = pv[i];
            };
            if (form == 0) {
#pragma unroll
                for (int i = 0; i < ITEMS; i++)
                    if (valid_at(i)) scatter(t_rank(digit(v[i])), i);
            } else if (form == 1) {
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const bool valid = valid_at(i);
                    const uint32_t dd = digit(v[i]);
                    const uint32_t dw = __shfl_sync(kFull, dd, 0);
                    if (__all_sync(kFull, !valid || dd == dw)) {
                        const uint32_t vm = FULL ? kFull : __ballot_sync(kFull, valid);
                        const uint32_t c = t_get(dw);
                        __syncwarp();
                        if (lane == 0) t_add(dw, __popc(vm));
                        if (valid) scatter(c + __popc(vm & ltj), i);
                        __syncwarp();
                    } else if (valid) {
                        scatter(t_rank(dd), i);
                    }
                }
            } else {
                uint32_t hb[NHOT];  // this warp's running slot of each hot digit
#pragma unroll
                for (int k = 0; k < NHOT; k++) hb[k] = hot[k] != 0xffffffffu ? t_get(hot[k]) : 0u;
                __syncwarp();
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const bool valid = valid_at(i);
                    const uint32_t dd = digit(v[i]);
                    uint32_t pos = 0;
                    bool h = false;
#pragma unroll
                    for (int k = 0; k < NHOT; k++) {
                        if (k < nh) {  // warp-uniform
                            const bool mine = valid && dd == hot[k];
                            const uint32_t m = __ballot_sync(kFull, mine);
                            if (mine) pos = hb[k] + __popc(m & ltj);
                            hb[k] += __popc(m);
                            h |= mine;
                        }
                    }
                    if (valid && !h) pos = t_rank(dd);
                    if (valid) scatter(pos, i);
                }
            }
            __syncwarp();
            // this warp's digit table: cleared for the next tile
            {
                uint4 *t4 = reinterpret_cast<uint4 *>(cw);
#pragma unroll
                for (int q = 0; q < TW / 4 / 32; q++) t4[q * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
            }

            // ------------------------------------------- decoupled look-back
            if (tid < (uint32_t)NT) {
                uint32_t excl[DPT];
#pragma unroll
                for (int j = 0; j < DPT; j++) excl[j] = 0u;
                if (!(AHS_OS2_ABL & 8) && tile > 0) {
                    uint32_t need = (1u << DPT) - 1u;  // digits without an inclusive predecessor yet
                    int jt = (int)tile - 1;
                    uint32_t spins = 0;
                    while (true) {
                        os2::Vec<DPT> st[kLookback];
                        const uint32_t *ps = status + (size_t)jt * BINS + d0;
                        if (jt >= kLookback - 1) {
#pragma unroll
                            for (int q = 0; q < kLookback; q++) st[q] = os2::ld_status<DPT>(ps - (size_t)q * BINS);
                        } else {
#pragma unroll
                            for (int q = 0; q < kLookback; q++) {
                                if (jt - q >= 0) {
                                    st[q] = os2::ld_status<DPT>(ps - (size_t)q * BINS);
                                } else {
#pragma unroll
                                    for (int j = 0; j < DPT; j++) st[q].w[j] = kFlagIncl;
                                }
                            }
                        }
                        int used = 0;
                        bool stop = false;
#pragma unroll
                        for (int q = 0; q < kLookback; q++) {
                            if (!stop) {
                                bool pub = true;
#pragma unroll
                                for (int j = 0; j < DPT; j++)
                                    pub &= !((need >> j) & 1u) || (st[q].w[j] & ~kCountMask) != 0u;
                                if (!pub) {
                                    stop = true;
                                } else {
#pragma unroll
                                    for (int j = 0; j < DPT; j++) {
                                        if ((need >> j) & 1u) {
                                            excl[j] += st[q].w[j] & kCountMask;
                                            if ((st[q].w[j] & ~kCountMask) == kFlagIncl) need &= ~(1u << j);
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
                            if (++spins > kLookbackSpinLimit) {
                                if (!a.fault) __trap();
                                atomicExch(a.fault, 1u);
                                break;
                            }
                            __nanosleep(64);
                        }
                    }
                    uint32_t sts[DPT];
#pragma unroll
                    for (int j = 0; j < DPT; j++) sts[j] = kFlagIncl | (excl[j] + tot[j]);
                    os2::st_status<DPT>(&status[(size_t)tile * BINS + d0], sts);
                }
#pragma unroll
                for (int j = 0; j < DPT; j++) s_gofs[d0 + j] = __ldg(&bucket_base[d0 + j]) + excl[j] - s_start[d0 + j];
            }
            __syncthreads();
            if (tid == 0) {
                const uint32_t nt = atomicAdd(tile_ticket, 1u);
                s_ticket[b ^ 1u] = nt;
                if (nt < ntiles && tma_ok && tile_full(nt)) {
                    fence_proxy_async();
                    issue(nt, b ^ 1u);
                }
            }

            // ------------------------------------------------------- write out
            auto emit = [&](uint32_t i, K x, [[maybe_unused]] V y) {
                const uint32_t o = s_gofs[digit(x)] + i;
                if constexpr (TOUT) x = (x + subv) ^ flip;
                keys_out[o] = x;
                if constexpr (KV) vals_out[o] = y;
            };
            if constexpr (FULL && BLOCK == 512) {
#pragma unroll
                for (int k = 0; k < ITEMS; k++) {
                    const uint32_t sl = ((k & 1) ? wo1 : wo0) + k * BLOCK;
                    V y = V(0);
                    if constexpr (KV) y = sv[sl];
                    emit(tid + k * BLOCK, sk[sl], y);
                }
            } else {
                for (uint32_t i = tid; i < tile_n; i += BLOCK) {
                    const uint32_t sp = i ^ ((i >> 5) & 31u);
                    V y = V(0);
                    if constexpr (KV) y = sv[sp];
                    emit(i, sk[sp], y);
                }
            }
        };
        if (full) tile_work(std::true_type{});
        else tile_work(std::false_type{});
        __syncthreads();
    }
}

template <bool KV, int BLOCK, int ITEMS, int MINB, int BITS = 8, typename K = uint32_t, typename V = uint32_t,
          int HOTCFG = kHotDefault>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep2(const PassArgsT<K, V> a)
{
    pdl_begin();
    // the other status region is cleared for the next pass at the end (as K6 does)
    auto clear_other = [&] {
        // (a next pass that the plan skips uses no statuses: its own launch clears for the one after)
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
    const K *keys_in = first ? a.keys_in : (from_out ? a.keys_out : a.keys_tmp);
    const V *vals_in = first ? a.vals_in : (from_out ? a.vals_out : a.vals_tmp);
    K *keys_out = to_out ? a.keys_out : a.keys_tmp;
    V *vals_out = to_out ? a.vals_out : a.vals_tmp;
    // the key transforms are identities for unsigned keys with min 0: treat them as such
    const bool tin = first && (a.flip != K(0) || a.sub != K(0));
    const bool tout = last && (a.flip != K(0) || a.sub != K(0));
    if (tin) {
        if (tout) onesweep2_body<KV, BLOCK, ITEMS, BITS, true, true, K, V, HOTCFG>(a, keys_in, vals_in, keys_out, vals_out, shift);
        else onesweep2_body<KV, BLOCK, ITEMS, BITS, true, false, K, V, HOTCFG>(a, keys_in, vals_in, keys_out, vals_out, shift);
    } else {
        if (tout) onesweep2_body<KV, BLOCK, ITEMS, BITS, false, true, K, V, HOTCFG>(a, keys_in, vals_in, keys_out, vals_out, shift);
        else onesweep2_body<KV, BLOCK, ITEMS, BITS, false, false, K, V, HOTCFG>(a, keys_in, vals_in, keys_out, vals_out, shift);
    }
    clear_other();
}

}  // namespace ahs
