// onesweep.cuh — K6: one stable 8-bit LSD digit pass, onesweep style
// (one read + one write of the keys per pass; §III.G,
// each pass a stable counting sort by one base-256 digit, Eq. 4).
//
// Persistent CTAs (two per SM).  A CTA takes tiles from an atomic ticket in
// increasing order; the ticket for its next tile is taken only once the
// current tile's inclusive prefix is published (a held-but-unstarted tile then
// waits on nothing but this CTA's write-out), and that tile's keys arrive by
// TMA bulk copy in the second shared-memory buffer during the write-out.
// Per tile:
//
//   early     keys (and values) into registers; each half-warp ("sub-warp",
//   counts    16 lanes) owns a contiguous segment of 16 x ITEMS keys and counts
//             its digits in a 256-word table with shared atomics (a warp whose
//             32 keys share one digit adds once: same-address atomics serialise).
//   publish   per digit: tile count -> status word (aggregate) for the
//             look-back of later tiles, before any ranking.
//   offsets   tile digit starts (scan over the 256 counts); each sub-warp table
//             is rewritten as {lane mask 0 | slot = digit start + earlier
//             sub-warps' count}.
//   rank +    per item every lane adds (1 << (16 + j)) + 1 to its digit's word,
//   scatter   reads it back (mask = its peers in this item, slot advanced by
//             their number) and clears the mask half: tile position = slot -
//             popc(peers at or above me).  Stable (items in order, lanes in
//             order), three shared-memory operations per key, no match.any
//             (~60 cycles per warp instruction on sm_100).  Keys (and values)
//             go straight to their tile position in shared memory.
//   look-back decoupled look-back over predecessor tiles (kLookback statuses
//             per round), inclusive status published.
//   write     consecutive tile slots of one digit -> consecutive global slots
//             (coalesced), output transform fused.
//
// The two half-warps of one warp read segments 16 * ITEMS apart (ITEMS odd),
// i.e. disjoint bank halves: key loads from shared memory are conflict-free.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace ahs {

// status[tile][digit] = flag << 30 | count (count < 2^30 > AHS_MAX_N)
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1u;
constexpr int kBins = 256;     // 8-bit digits
#ifndef AHS_LOOKBACK
#define AHS_LOOKBACK 8
#endif
constexpr int kLookback = AHS_LOOKBACK;  // predecessor statuses loaded per look-back round (B200: 8 beats 16, 32)
#ifdef AHS_PHASE_STATS
// development instrumentation (tools/passbench.cu -DAHS_PHASE_STATS): cycles
// per tile phase and look-back rounds, seen by thread 0 of each CTA
__device__ unsigned long long g_phase_cycles[8];
__device__ unsigned long long g_lb_probe[4];  // look-backs, rounds, cycles in rounds, empty rounds
#define PHASE_MARK(k)                                                       \
    do {                                                                    \
        if (threadIdx.x == 0) {                                             \
            const long long t_ = clock64();                                 \
            atomicAdd(&g_phase_cycles[k], (unsigned long long)(t_ - t_ph)); \
            t_ph = t_;                                                      \
        }                                                                   \
    } while (0)
#else
#define PHASE_MARK(k) \
    do {              \
    } while (0)
#endif
#ifdef AHS_LB_STATS
__device__ unsigned long long g_lb_stats[4];  // tiles, rounds, empty rounds, statuses consumed
#endif

__device__ __forceinline__ uint32_t digit8(uint32_t v, uint32_t shift)
{
    // any bit offset: the bucket-local GENERAL plan runs digits at the feature-bin shift
    return (v >> shift) & 255u;
}

// 64-bit keys (NEXT-3): digit at bit `shift` (a multiple of 8, < 64)
__device__ __forceinline__ uint32_t digit8(uint64_t v, uint32_t shift)
{
    return (uint32_t)(v >> shift) & 255u;
}

// Shared-memory index of tile slot i in the reordered tile: XOR-swizzled so
// that 32 consecutive slots stay conflict-free (write-out) while slots 32
// apart land in different banks (an ascending input puts exactly 32 keys per
// digit into an 8192-key tile: its scatter would otherwise hit one bank).
__device__ __forceinline__ uint32_t swz(uint32_t i) { return i ^ ((i >> 5) & 31u); }
// The same for 64-bit slots (16 per 128-byte bank row): 16 consecutive slots (one
// half-warp phase of a 64-bit access) stay conflict-free.
__device__ __forceinline__ uint32_t swz64(uint32_t i) { return i ^ ((i >> 4) & 15u); }

// Key-value passes over 32-bit keys and values (ordered ranking) reorder each pair as
// one packed 64-bit slot (value << 32 | key): one scatter store and one write-out load
// per pair instead of two.  A tile buffer then holds its keys and values side by side
// ([b][keys TILE | values TILE]) so that the packed slots reuse its 8 * TILE bytes.
#ifndef AHS_K6_PACK
#define AHS_K6_PACK 1
#endif

// RANK: kRankMasked  16-lane sub-warps, {lane mask | slot} words: atomic add,
//                    read-back, mask clear (makes no assumption about the order
//                    in which the lanes of one atomic instruction are served).
//       kRankOrdered whole warps, plain slot counters: one atomic add with
//                    return per key IS the rank.  Correct only on hardware that
//                    serves the same-address lanes of one shared-memory atomic
//                    instruction in ascending lane order (B200 does: 11.6e9 of
//                    11.6e9 in tools/atomorder.cu); the CUDA model leaves that
//                    order unspecified, so the host selects this mode only after
//                    a self-test of the property on the device (ahs_api.cu).
constexpr int kRankMasked = 0;
constexpr int kRankOrdered = 1;

template <bool KV, int BLOCK, int ITEMS, int RANK = kRankMasked, typename K = uint32_t, typename V = uint32_t>
struct Onesweep {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kGroupLanes = RANK == kRankOrdered ? 32 : 16;  // lanes sharing one digit table
    static constexpr int kSub = BLOCK / kGroupLanes;                     // digit tables per CTA
    static constexpr int kTile = BLOCK * ITEMS;
    static constexpr int kSeg = kGroupLanes * ITEMS;  // keys per table owner
    static constexpr int kTPD = BLOCK / kBins;  // threads per digit in the per-tile scans
    static_assert(RANK == kRankOrdered || ITEMS % 2 == 1,
                  "odd ITEMS: the half-warps of a warp read disjoint bank halves");
    static_assert(BLOCK * ITEMS < 65536, "16-bit slot field");
    static_assert(BLOCK >= 256 && BLOCK <= 512 && BLOCK % 128 == 0, "256, 384 or 512 threads");
    static_assert((kTile * 4) % 16 == 0, "TMA tile size");
    static constexpr size_t kBufK = (size_t)kTile * sizeof(K);           // keys: 4 or 8 bytes
    static constexpr size_t kBuf = (size_t)kTile * sizeof(V);            // values: 4 or 8 bytes
    static constexpr size_t kOffK = 0;                                   // keys   [2][TILE]
    static constexpr size_t kOffV = kOffK + 2 * kBufK;                   // values [2][TILE]
    static constexpr size_t kOffCnt = kOffV + (KV ? 2 * kBuf : 0);       // digit tables [SUB][256]
    static constexpr size_t kOffAux = kOffCnt + (size_t)kSub * kBins * 4;
    // aux: part[2][256], start[256], gofs[256], wsum[8]
    static constexpr size_t kSmem = kOffAux + (size_t)(4 * kBins + 8) * 4;
};

// Device pass plan word (K5): kPassSkip, or (digit shift << 16) | (executed index << 8) | executed count.
constexpr uint32_t plan_word(uint32_t shift, uint32_t e, uint32_t m) { return (shift << 16) | (e << 8) | m; }

// One digit pass of a chain of `npasses` LSD passes.  Buffers: the chain reads
// `keys_in` (first executed pass, input transform v = (key ^ flip) - sub) and
// ping-pongs between `keys_tmp` and `keys_out` so that the last executed pass
// (output transform key = (v + sub) ^ flip) lands in `keys_out`.  With a
// device plan (K5, NEXT-1 trivial-pass skipping) a pass whose digit is the
// same for every key is an identity permutation: its launch returns at once,
// and the executed passes are renumbered 0 .. m-1 (plan word: exec index << 8
// | m, or kPassSkip).  Without a plan, pass p is executed pass p of npasses.
constexpr uint32_t kPassSkip = 0xffffffffu;
template <typename K, typename V = uint32_t>
struct PassArgsT {
    const K *keys_in;
    const V *vals_in;
    K *keys_out;
    V *vals_out;
    K *keys_tmp;
    V *vals_tmp;
    uint32_t n, pass, npasses, shift;
    K flip, sub;
    const uint32_t *bucket_base;  // this pass's 256 digit bases
    uint32_t *status, *ticket;    // this pass's look-back statuses and tile ticket (zeroed)
    const uint32_t *plan;         // nullptr: no skipping
    uint32_t *status_clear;       // the other status region: zeroed at the end of this pass for the next
    uint32_t clear_words;         //   (passes alternate between two regions; 0: nothing to clear)
    uint32_t *fault;              // set to 1 when a look-back gives up (nullptr: __trap instead)
};

// Look-back polls before a pass gives up on an unpublished predecessor (each empty round
// sleeps >= 64 ns: > 17 s).  A predecessor CTA can be descheduled for a long time (time
// slicing, MPS, a debugger), so the bound is far above any legitimate wait; when it is hit
// the pass sets *fault (the host reports AHS_ECUDA) and finishes instead of trapping, which
// would kill the context for every stream of the process.
constexpr uint32_t kLookbackSpinLimit = 1u << 28;
using PassArgs = PassArgsT<uint32_t>;

// K: uint32_t (32-bit keys) or uint64_t (64-bit keys, NEXT-3); V: the value type (uint32_t,
// or uint64_t for 64-bit payloads, NEXT-3)
template <bool KV, int BLOCK, int ITEMS, int MINB, int RANK = kRankMasked, typename K = uint32_t,
          typename V = uint32_t>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep(const PassArgsT<K, V> a)
{
    pdl_begin();
    // the previous pass is complete (pdl_begin): its status region is free and is cleared for the
    // pass after this one -- by each CTA once its tiles are done (the tail of the pass), or at once
    // when this pass is skipped
    auto clear_other = [&] {
        // (a next pass that the plan skips uses no statuses: its own launch clears for the one after)
        if (a.plan && a.plan[a.pass + 1] == kPassSkip) return;
        for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < a.clear_words; i += gridDim.x * BLOCK)
            a.status_clear[i] = 0u;
    };
    // ---- this pass's place in the chain (and its digit's bit offset, from the plan when there is one)
    uint32_t e = a.pass, m = a.npasses, shift = a.shift;
    if (a.plan) {
        const uint32_t w = a.plan[a.pass];
        if (w == kPassSkip) {  // constant digit (or a pass the plan does not use): identity
            clear_other();
            return;
        }
        e = (w >> 8) & 255u;
        m = w & 255u;
        shift = w >> 16;
    }
    const bool first = e == 0, last = e + 1 == m;
    const bool to_out = ((m - 1 - e) & 1u) == 0;        // destination parity: the last lands in out
    const bool from_out = !first && !to_out;             // source = the previous pass's destination
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

    using C = Onesweep<KV, BLOCK, ITEMS, RANK, K, V>;
    constexpr int TILE = C::kTile, SEG = C::kSeg, GL = C::kGroupLanes;
    constexpr bool ORDERED = RANK == kRankOrdered;
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

    constexpr bool PK = AHS_K6_PACK && KV && ORDERED && sizeof(K) == 4 && sizeof(V) == 4;
    // tile buffer b: keys and values (PK: side by side, [b][keys | values])
    auto kbuf = [&](uint32_t b) -> K * { return PK ? s_kb + b * 2 * TILE : s_kb + b * TILE; };
    auto vbuf = [&](uint32_t b) -> V * {
        return PK ? reinterpret_cast<V *>(s_kb) + b * 2 * TILE + TILE : s_vb + b * TILE;
    };
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t h = ORDERED ? 0u : lane >> 4, j = ORDERED ? lane : lane & 15u;
    const uint32_t sub = ORDERED ? warp : warp * 2u + h;
    const uint32_t ntiles = (n + TILE - 1) / TILE;
    const uint32_t ltj = ORDERED ? lanemask_lt() : (1u << j) - 1u;  // lanes before me in my group

    auto tile_full = [&](uint32_t t) { return (uint64_t)(t + 1) * TILE <= n; };
    auto issue = [&](uint32_t t, uint32_t b) {  // thread 0
        const uint32_t kbytes = (uint32_t)(TILE * sizeof(K)), vbytes = (uint32_t)(TILE * sizeof(V));
        mbar_expect_tx(&s_bar[b], kbytes + (KV ? vbytes : 0u));
        tma_load_1d(kbuf(b), keys_in + (size_t)t * TILE, kbytes, &s_bar[b]);
        if constexpr (KV) tma_load_1d(vbuf(b), vals_in + (size_t)t * TILE, vbytes, &s_bar[b]);
    };

    // skewed digit distribution (a digit holds > 1/16 of the keys): enable the
    // warp-uniform fast path (same-address shared atomics serialise)
    __shared__ uint32_t s_skew;
    if (tid == 0) s_skew = 0u;
    __syncthreads();
    if (tid < kBins) {
        const uint32_t hi = tid == kBins - 1 ? n : __ldg(&bucket_base[tid + 1]);
        if (hi - __ldg(&bucket_base[tid]) > n / 16u) s_skew = 1u;
    }
    for (int i = tid; i < C::kSub * kBins / 4; i += BLOCK)
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
    uint32_t phase = 0;  // bit b: parity of buffer b's next completion
#ifdef AHS_PHASE_STATS
    long long t_ph = clock64();
#endif
    for (uint32_t iter = 0;; iter++) {
        const uint32_t b = iter & 1u;
        const uint32_t tile = s_ticket[b];
        if (tile >= ntiles) break;
        const uint32_t tile_base = tile * (uint32_t)TILE;
        const uint32_t tile_n = min((uint32_t)TILE, n - tile_base);
        const bool full = tile_n == (uint32_t)TILE;
        K *sk = kbuf(b);
        V *sv = vbuf(b);
        [[maybe_unused]] uint64_t *s_slot = reinterpret_cast<uint64_t *>(sk);  // PK: packed pairs
        if (tma_ok && full) {
            mbar_wait(&s_bar[b], (phase >> b) & 1u);
            PHASE_MARK(0);
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
            // uniform-digit fast path for this warp and tile: on when the pass is
            // skewed, or when the warp's first 32 keys share one digit (sorted
            // runs); decided once per warp, a warp-uniform runtime branch
            bool wskew = skew;
            // --------------------------------------------- early counts
            // keys (and values) into registers; per sub-warp digit counts
            K v[ITEMS];
            [[maybe_unused]] V pv[KV ? ITEMS : 1];
            uint32_t *cw = s_cnt + sub * kBins;
            const uint32_t sbase = sub * SEG + j;
    #pragma unroll
            for (int it = 0; it < ITEMS; it++) {
                const uint32_t idx = sbase + it * GL;
                const bool valid = FULL || idx < tile_n;
                v[it] = ((valid ? sk[idx] : K(0)) ^ in_flip) - in_sub;
                if constexpr (KV) pv[it] = valid ? sv[idx] : V(0);
                const uint32_t d = digit8(v[it], shift);
                if (it == 0 && !wskew) wskew = __all_sync(kFull, d == __shfl_sync(kFull, d, 0));
                // the count atomic returns nothing: the lanes of one instruction that hit the same
                // word are merged by the hardware, so warp-uniform digits need no special path here
                // (only the returning rank atomic below serialises them)
                if (valid) atomicAdd(&cw[d], 1u);
            }
            __syncthreads();
            PHASE_MARK(1);

            // ------------------ per-digit totals, publish aggregate, tile scan
            const uint32_t d = tid & (kBins - 1), part = tid / kBins;
            constexpr int SPP = C::kSub / C::kTPD;  // sub-warps per thread
            uint32_t psum = 0;
            if (C::kTPD == 2 || tid < kBins) {
    #pragma unroll 8
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
            PHASE_MARK(2);
            // sub-warp digit offsets in the tile (digit start + earlier sub-warps)
            if (C::kTPD == 2 || tid < kBins) {
                uint32_t run = s_start[d] + (part ? s_part[d] : 0u);
    #pragma unroll 8
                for (int s = 0; s < SPP; s++) {
                    uint32_t *p = &s_cnt[(part * SPP + s) * kBins + d];
                    const uint32_t c = *p;
                    *p = run;
                    run += c;
                }
            }
            __syncthreads();
            PHASE_MARK(3);

            // ------------------------------------- rank + scatter in digit order
            // word = {bit 16+j: lane j has this digit in this item | low 16: next slot}
    #pragma unroll
            for (int it = 0; it < ITEMS; it++) {
                const uint32_t idx = sbase + it * GL;
                const bool valid = FULL || idx < tile_n;
                const uint32_t dd = digit8(v[it], shift);
                uint32_t pos = 0;
                bool done = false;
                if (wskew) {
                    const uint32_t d0 = __shfl_sync(kFull, dd, 0);
                    if (__all_sync(kFull, !valid || dd == d0)) {
                        const uint32_t vm = FULL ? kFull : __ballot_sync(kFull, valid);
                        const uint32_t gm = ORDERED ? vm : (vm >> (h * 16u)) & 0xffffu;
                        const uint32_t c = cw[d0];
                        pos = c + __popc(gm & ltj);
                        __syncwarp();
                        if (j == 0) cw[d0] = c + __popc(gm);
                        done = true;
                    }
                }
                if (!done) {
                    if constexpr (ORDERED) {
                        // lanes of this instruction are served in lane order (self-tested)
                        if (valid) pos = atomicAdd(&cw[dd], 1u);
                    } else {
                        if (valid) atomicAdd(&cw[dd], (1u << (16u + j)) + 1u);
                        __syncwarp();
                        const uint32_t w = cw[dd];
                        __syncwarp();
                        if (valid) reinterpret_cast<uint16_t *>(cw + dd)[1] = 0;
                        pos = (w & 0xffffu) - __popc(w >> (16u + j));
                    }
                }
                if (valid) {
                    if constexpr (PK) {
                        s_slot[swz64(pos)] = (uint64_t)pv[it] << 32 | v[it];
                    } else {
                        sk[swz(pos)] = v[it];
                        if constexpr (KV) sv[swz(pos)] = pv[it];
                    }
                }
                __syncwarp();
            }
            // this warp's digit tables are no longer needed: clear for the next tile
            {
                constexpr int TPW = 32 / GL;  // tables per warp
                uint4 *t4 = reinterpret_cast<uint4 *>(s_cnt + warp * TPW * kBins);
    #pragma unroll
                for (int q = 0; q < TPW * kBins / 4 / 32; q++) t4[q * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
            }

            PHASE_MARK(4);
            // ------------------------------------------- decoupled look-back
            // kLookback predecessor statuses per round, consumed newest-first: AGG
            // counts accumulate, the first INCL ends the walk, an unpublished one is
            // re-read next round.  Tile -1 is INCL 0.
            if (tid < kBins) {
                uint32_t excl = 0;
                if (tile > 0) {
                    int jt = (int)tile - 1;
                    uint32_t spins = 0;
#ifdef AHS_PHASE_STATS
                    const long long t_lb0 = clock64();
                    uint32_t n_rounds = 0, n_empty = 0;
#endif
                    while (true) {
#ifdef AHS_PHASE_STATS
                        n_rounds++;
#endif
                        uint32_t st[kLookback];
                        if (jt >= kLookback - 1) {  // the whole window exists: one base, immediate offsets
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
#ifdef AHS_LB_STATS
                        atomicAdd(&g_lb_stats[1], 1ull);
                        atomicAdd(&g_lb_stats[3], (unsigned long long)used);
                        if (used == 0) atomicAdd(&g_lb_stats[2], 1ull);
#endif
                        if (fin) break;
                        jt -= used;
#ifdef AHS_PHASE_STATS
                        n_empty += used == 0;
#endif
                        if (used == 0) {
                            // predecessors hold earlier tickets and publish before they wait
                            if (++spins > kLookbackSpinLimit) {
                                if (!a.fault) __trap();
                                atomicExch(a.fault, 1u);
                                break;
                            }
                            __nanosleep(64);
                        }
                    }
                    st_relaxed(&status[(size_t)tile * kBins + d], kFlagIncl | (excl + total));
#ifdef AHS_PHASE_STATS
                    if (tid == 0) {
                        atomicAdd(&g_lb_probe[0], 1ull);
                        atomicAdd(&g_lb_probe[1], (unsigned long long)n_rounds);
                        atomicAdd(&g_lb_probe[2], (unsigned long long)(clock64() - t_lb0));
                        atomicAdd(&g_lb_probe[3], (unsigned long long)n_empty);
                    }
#endif
#ifdef AHS_LB_STATS
                    atomicAdd(&g_lb_stats[0], 1ull);
#endif
                }
                s_gofs[d] = __ldg(&bucket_base[d]) + excl - s_start[d];
            }
            __syncthreads();
            PHASE_MARK(5);
            // Next tile: its ticket is taken only now, after this tile's inclusive
            // prefix is published, so a tile whose ticket is held but not yet
            // started never waits on anything but this CTA's write-out (taking it
            // earlier chains the look-backs of different CTAs into convoys).  Its
            // keys arrive in the other buffer (free: the last tile ended with a
            // barrier) during the write-out below.
            if (tid == 0) {
                const uint32_t nt = atomicAdd(tile_ticket, 1u);
                s_ticket[b ^ 1u] = nt;
                if (nt < ntiles && tma_ok && tile_full(nt)) {
                    fence_proxy_async();
                    issue(nt, b ^ 1u);
                }
            }

            // ------------------------------------------------------- write out
            if constexpr (PK) {
                const uint32_t lim = FULL ? (uint32_t)TILE : tile_n;
    #pragma unroll 4
                for (uint32_t i = tid; i < lim; i += BLOCK) {
                    const uint64_t x = s_slot[swz64(i)];
                    const K xk = (K)(uint32_t)x;
                    const uint32_t o = s_gofs[digit8(xk, shift)] + i;
                    keys_out[o] = (xk + out_add) ^ out_flip;
                    vals_out[o] = (V)(uint32_t)(x >> 32);
                }
            } else if constexpr (FULL) {
    #pragma unroll 5
                for (int i = tid; i < TILE; i += BLOCK) {
                    const K x = sk[swz(i)];
                    const uint32_t o = s_gofs[digit8(x, shift)] + i;
                    keys_out[o] = (x + out_add) ^ out_flip;
                    if constexpr (KV) vals_out[o] = sv[swz(i)];
                }
            } else {
                for (uint32_t i = tid; i < tile_n; i += BLOCK) {
                    const K x = sk[swz(i)];
                    const uint32_t o = s_gofs[digit8(x, shift)] + i;
                    keys_out[o] = (x + out_add) ^ out_flip;
                    if constexpr (KV) vals_out[o] = sv[swz(i)];
                }
            }
        };
        if (full) tile_work(std::true_type{});
        else tile_work(std::false_type{});
        __syncthreads();
        PHASE_MARK(6);
    }
    clear_other();
}

// Self-test of the hardware property kRankOrdered relies on: the lanes of one
// shared-memory atomicAdd instruction that hit the same address are served in
// ascending lane order, so the returned old values are lane-ordered ranks.
// Same source pattern as the ranking loops (per-warp 256-word tables, items in
// sequence separated by __syncwarp, the atomic's return value used), with digit
// collision rates from "all 32 lanes on one word" to "spread over 256 words",
// and with the active-lane masks the kernels issue: the full warp (K6 full
// tiles, K9r, whose idle lanes hit a dummy word), a prefix of the lanes (K6's
// partial last tile: `if (valid) atomicAdd`), a suffix and scattered lanes.
// Expected ranks come from match.any (slow but independent).  *bad counts
// violations.  (tests/test_sass_rank.py checks that this kernel and the ranking
// kernels compile the rank site to the same ATOMS.ADD-with-return form.)
__device__ __forceinline__ uint32_t selftest_hash(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__global__ void __launch_bounds__(512)
    k_lane_order_selftest(uint32_t *__restrict__ bad, int items)
{
    __shared__ uint32_t tab[16][kBins];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16 * kBins; i += blockDim.x) (&tab[0][0])[i] = 0u;
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    uint32_t nbad = 0;
    for (int it = 0; it < items; it++) {
        const uint32_t r = selftest_hash((blockIdx.x * blockDim.x + threadIdx.x) * 977u + it * 0x9e3779b9u);
        const uint32_t mask = (1u << (it % 9)) - 1u;  // 1 .. 256 distinct words
        const uint32_t dd = (r & mask) * (kBins / (mask + 1u));
        // active lanes of this item (warp-uniform): full, prefix, suffix, scattered
        const uint32_t h = selftest_hash(blockIdx.x * 7919u + warp * 104729u + (uint32_t)it);
        const uint32_t m = 1u + h % 31u;  // 1 .. 31
        const uint32_t kind = (uint32_t)(it / 9) % 4u;
        const uint32_t act = kind == 0 ? kFull
                           : kind == 1 ? (1u << m) - 1u                   // lanes < m
                           : kind == 2 ? ~((1u << m) - 1u)                // lanes >= m
                                       : (selftest_hash(h) | 1u);         // scattered, lane 0 active
        if ((act >> lane) & 1u) {
            const uint32_t pos = atomicAdd(&tab[warp][dd], 1u);
            const uint32_t peers = __match_any_sync(act, dd);
            const uint32_t base = __shfl_sync(act, pos, __ffs(peers) - 1);
            nbad += pos != base + __popc(peers & lt);
        }
        __syncwarp();
    }
    nbad = __reduce_add_sync(kFull, nbad);
    if (lane == 0 && nbad) atomicAdd(bad, nbad);
}

}  // namespace ahs
