// onesweep2.cuh — K6 v2: the onesweep digit pass of onesweep.cuh (one stable
// 8-bit LSD digit pass: PAPER.md §III.G, each pass a stable
// counting sort by one base-256 digit, Eq. 4), rewritten for fewer
// instructions per key.  Same algorithm, data layout, statuses and pass
// chain as K6 (ordered ranking only: the masked fallback stays in K6):
//
//   * the tile loop is instantiated per (input transform, output transform):
//     only the first executed pass of a chain maps key -> (key ^ flip) - min,
//     only the last maps back; middle passes move keys untouched.  The
//     variant is picked once per launch from the device pass plan (NEXT-1).
//   * the count and rank loops come in two forms chosen once per warp and
//     tile: the plain loop (one shared atomic per key, no warp votes) and the
//     warp-uniform-digit loop (skewed passes, sorted runs);
//   * each warp's digit table is addressed from a per-warp base pointer;
//   * the write-out reads the XOR-swizzled reorder buffer from two
//     precomputed per-thread bases (512-thread CTAs: the swizzle of slot
//     tid + k * 512 only depends on k's parity), one LDS per key.
#pragma once

#include "onesweep.cuh"

// development ablations (tools/passbench.cu only; wrong results): bit 0 no count atomics,
// bit 1 scatter to the load slot, bit 2 rank by table read, bit 3 no look-back, bit 4 no global stores
#ifndef AHS_OS2_ABL
#define AHS_OS2_ABL 0
#endif

namespace ahs {

template <bool KV, int BLOCK, int ITEMS, typename K = uint32_t, typename V = uint32_t>
struct Onesweep2 {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * ITEMS;
    static constexpr int kSeg = 32 * ITEMS;      // keys per warp (its digit table)
    static constexpr int kTPD = BLOCK / kBins;   // threads per digit in the per-tile scans (1 or 2)
    static_assert(BLOCK == 256 || BLOCK == 384 || BLOCK == 512, "256, 384 or 512 threads");
    static_assert(kTile < 65536, "tile positions");
    static_assert((kTile * sizeof(K)) % 16 == 0 && (kTile * sizeof(V)) % 16 == 0, "TMA tile size");
    static constexpr size_t kBufK = (size_t)kTile * sizeof(K);
    static constexpr size_t kBufV = (size_t)kTile * sizeof(V);
    static constexpr size_t kOffK = 0;
    static constexpr size_t kOffV = kOffK + 2 * kBufK;
    static constexpr size_t kOffCnt = kOffV + (KV ? 2 * kBufV : 0);
    static constexpr size_t kOffAux = kOffCnt + (size_t)kWarps * kBins * 4;
    // aux: part[2][256], start[256], gofs[256], wsum[8]
    static constexpr size_t kSmem = kOffAux + (size_t)(4 * kBins + 8) * 4;
};


template <bool KV, int BLOCK, int ITEMS, int MINB, typename K = uint32_t, typename V = uint32_t>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep2(const PassArgsT<K, V> a);

template <bool KV, int BLOCK, int ITEMS, bool TIN, bool TOUT, typename K, typename V>
__device__ __forceinline__ void onesweep2_body(const PassArgsT<K, V> &a, const K *__restrict__ keys_in,
                                               const V *__restrict__ vals_in, K *__restrict__ keys_out,
                                               V *__restrict__ vals_out)
{
    using C = Onesweep2<KV, BLOCK, ITEMS, K, V>;
    constexpr int TILE = C::kTile, SEG = C::kSeg, NWARP = C::kWarps;
    constexpr uint32_t KB = sizeof(K), VB = sizeof(V);
    const uint32_t n = a.n, shift = a.shift;
    const K flip = a.flip, subv = a.sub;
    const uint32_t *__restrict__ bucket_base = a.bucket_base;
    uint32_t *__restrict__ status = a.status;
    uint32_t *__restrict__ tile_ticket = a.ticket;
    const uint32_t tma_ok = (((uintptr_t)keys_in & 15u) == 0) && (!KV || ((uintptr_t)vals_in & 15u) == 0);

    extern __shared__ __align__(128) uint8_t smem[];
    K *s_kb = reinterpret_cast<K *>(smem + C::kOffK);
    V *s_vb = reinterpret_cast<V *>(smem + C::kOffV);
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(smem + C::kOffCnt);
    uint32_t *s_part = reinterpret_cast<uint32_t *>(smem + C::kOffAux);
    uint32_t *s_start = s_part + 2 * kBins;
    uint32_t *s_gofs = s_start + kBins;
    uint32_t *s_wsum = s_gofs + kBins;
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_ticket[2];
    __shared__ uint32_t s_skew;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t ntiles = (n + TILE - 1) / TILE;
    const uint32_t ltj = lanemask_lt();
    uint32_t *const cw = s_cnt + warp * kBins;  // this warp's digit table
    const uint32_t dsel = 0x4440u | (shift >> 3);           // PRMT selector of the digit byte (32-bit keys)

    auto digit = [&](K v) -> uint32_t {
        if constexpr (sizeof(K) == 4) return __byte_perm((uint32_t)v, 0u, dsel);
        else return (uint32_t)(v >> shift) & 255u;
    };
    auto tile_full = [&](uint32_t t) { return (uint64_t)(t + 1) * TILE <= n; };
    auto issue = [&](uint32_t t, uint32_t b) {
        const uint32_t kbytes = (uint32_t)(TILE * KB), vbytes = (uint32_t)(TILE * VB);
        mbar_expect_tx(&s_bar[b], kbytes + (KV ? vbytes : 0u));
        tma_load_1d(s_kb + b * TILE, keys_in + (size_t)t * TILE, kbytes, &s_bar[b]);
        if constexpr (KV) tma_load_1d(s_vb + b * TILE, vals_in + (size_t)t * TILE, vbytes, &s_bar[b]);
    };

    if (tid == 0) s_skew = 0u;
    __syncthreads();
    if (tid < kBins) {
        const uint32_t hi = tid == kBins - 1 ? n : __ldg(&bucket_base[tid + 1]);
        if (hi - __ldg(&bucket_base[tid]) > n / 16u) s_skew = 1u;
    }
    for (int i = tid; i < NWARP * kBins / 4; i += BLOCK)
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
            // warp-uniform-digit path: skewed pass, or this warp's first 32 keys share a digit
            bool wsk = skew;
            {
                const uint32_t idx = sbase;
                const bool valid = FULL || idx < tile_n;
                K x = valid ? sk[idx] : K(0);
                if constexpr (TIN) x = (x ^ flip) - subv;
                const uint32_t d = digit(x);
                if (!wsk) wsk = __all_sync(kFull, !valid || d == __shfl_sync(kFull, d, 0));
            }
            // --------------------------------------------- early counts
            if (!wsk) {
                // all loads first: the table atomics may alias the tile buffer for the compiler
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const uint32_t idx = sbase + i * 32;
                    const bool valid = FULL || idx < tile_n;
                    K x = (FULL || valid) ? sk[idx] : K(0);
                    if constexpr (TIN) x = (x ^ flip) - subv;
                    v[i] = x;
                    if constexpr (KV) pv[i] = (FULL || valid) ? sv[idx] : V(0);
                }
#pragma unroll
                for (int i = 0; i < ITEMS; i++)
                    if (!(AHS_OS2_ABL & 1) && (FULL || sbase + i * 32 < tile_n)) atomicAdd(&cw[digit(v[i])], 1u);
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const uint32_t idx = sbase + i * 32;
                    const bool valid = FULL || idx < tile_n;
                    K x = (FULL || valid) ? sk[idx] : K(0);
                    if constexpr (TIN) x = (x ^ flip) - subv;
                    v[i] = x;
                    if constexpr (KV) pv[i] = (FULL || valid) ? sv[idx] : V(0);
                    const uint32_t d = digit(x);
                    const uint32_t d0 = __shfl_sync(kFull, d, 0);
                    if (__all_sync(kFull, !valid || d == d0)) {
                        const uint32_t vm = FULL ? kFull : __ballot_sync(kFull, valid);
                        if (lane == 0) cw[d0] += __popc(vm);
                        __syncwarp();
                    } else if (FULL || valid) {
                        atomicAdd(&cw[d], 1u);
                    }
                }
            }
            __syncthreads();

            // ------------------ per-digit totals, publish aggregate, tile scan
            const uint32_t d = tid & (kBins - 1), part = tid / kBins;
            constexpr int SPP = NWARP / C::kTPD;
            uint32_t psum = 0;
            if (C::kTPD == 2 || tid < kBins) {
#pragma unroll
                for (int s = 0; s < SPP; s++) psum += s_cnt[(part * SPP + s) * kBins + d];
            }
            if constexpr (C::kTPD == 2) {
                s_part[part * kBins + d] = psum;
                __syncthreads();
            }
            uint32_t total = 0;
            if (tid < kBins) {
                total = C::kTPD == 2 ? s_part[d] + s_part[kBins + d] : psum;
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
                s_start[d] = before + incl - total;
            }
            __syncthreads();
            // per-warp digit offsets in the tile (digit start + earlier warps' counts)
            if (C::kTPD == 2 || tid < kBins) {
                uint32_t run = s_start[d] + (part ? s_part[d] : 0u);
#pragma unroll
                for (int s = 0; s < SPP; s++) {
                    uint32_t *p = &s_cnt[(part * SPP + s) * kBins + d];
                    const uint32_t c = *p;
                    *p = run;
                    run += c;
                }
            }
            __syncthreads();

            // ------------------------------------- rank + scatter in digit order
            auto scatter = [&](uint32_t pos, int i) {
                if (AHS_OS2_ABL & 2) pos = sbase + i * 32;
                const uint32_t sp = pos ^ ((pos >> 5) & 31u);
                sk[sp] = v[i];
                if constexpr (KV) sv[sp] = pv[i];
            };
            if (!wsk) {
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const bool valid = FULL || sbase + i * 32 < tile_n;
                    if (FULL || valid) scatter((AHS_OS2_ABL & 4) ? cw[digit(v[i])] + lane : atomicAdd(&cw[digit(v[i])], 1u), i);  // lane order (self-tested)
                }
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const bool valid = FULL || sbase + i * 32 < tile_n;
                    const uint32_t dd = digit(v[i]);
                    const uint32_t d0 = __shfl_sync(kFull, dd, 0);
                    if (__all_sync(kFull, !valid || dd == d0)) {
                        const uint32_t vm = FULL ? kFull : __ballot_sync(kFull, valid);
                        const uint32_t c = cw[d0];
                        __syncwarp();
                        if (lane == 0) cw[d0] = c + __popc(vm);
                        if (FULL || valid) scatter(c + __popc(vm & ltj), i);
                        __syncwarp();
                    } else if (FULL || valid) {
                        scatter(atomicAdd(&cw[dd], 1u), i);
                    }
                }
            }
            // this warp's digit table: cleared for the next tile
            {
                uint4 *t4 = reinterpret_cast<uint4 *>(s_cnt + warp * kBins);
#pragma unroll
                for (int q = 0; q < kBins / 4 / 32; q++) t4[q * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
            }

            // ------------------------------------------- decoupled look-back
            if (tid < kBins) {
                uint32_t excl = 0;
                if (!(AHS_OS2_ABL & 8) && tile > 0) {
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
                s_gofs[d] = __ldg(&bucket_base[d]) + excl - s_start[d];
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
                if (!(AHS_OS2_ABL & 16) || x == 0x12345u) keys_out[o] = x;
                if constexpr (KV) vals_out[o] = y;
            };
            if constexpr (FULL && BLOCK == 512) {
#pragma unroll
                for (int k = 0; k < ITEMS; k++) {
                    const uint32_t sl = ((k & 1) ? wo1 : wo0) + k * BLOCK;
                    const K x = sk[sl];
                    V y = V(0);
                    if constexpr (KV) y = sv[sl];
                    emit(tid + k * BLOCK, x, y);
                }
            } else {
                for (uint32_t i = tid; i < tile_n; i += BLOCK) {
                    const uint32_t sp = i ^ ((i >> 5) & 31u);
                    const K x = sk[sp];
                    V y = V(0);
                    if constexpr (KV) y = sv[sp];
                    emit(i, x, y);
                }
            }
        };
        if (full) tile_work(std::true_type{});
        else tile_work(std::false_type{});
        __syncthreads();
    }
}

template <bool KV, int BLOCK, int ITEMS, int MINB, typename K, typename V>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep2(const PassArgsT<K, V> a)
{
    pdl_begin();
    for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < a.clear_words; i += gridDim.x * BLOCK)
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
    const K *keys_in = first ? a.keys_in : (from_out ? a.keys_out : a.keys_tmp);
    const V *vals_in = first ? a.vals_in : (from_out ? a.vals_out : a.vals_tmp);
    K *keys_out = to_out ? a.keys_out : a.keys_tmp;
    V *vals_out = to_out ? a.vals_out : a.vals_tmp;
    // the key transforms are identities for uint32 keys with min 0: treat them as such
    const bool tin = first && (a.flip != K(0) || a.sub != K(0));
    const bool tout = last && (a.flip != K(0) || a.sub != K(0));
    if (tin) {
        if (tout) onesweep2_body<KV, BLOCK, ITEMS, true, true>(a, keys_in, vals_in, keys_out, vals_out);
        else onesweep2_body<KV, BLOCK, ITEMS, true, false>(a, keys_in, vals_in, keys_out, vals_out);
    } else {
        if (tout) onesweep2_body<KV, BLOCK, ITEMS, false, true>(a, keys_in, vals_in, keys_out, vals_out);
        else onesweep2_body<KV, BLOCK, ITEMS, false, false>(a, keys_in, vals_in, keys_out, vals_out);
    }
}

}  // namespace ahs
