// ahs_api.cu — host side of libahs.so: argument validation, workspace
// carving, the FSM, pass planning and the kernel launch sequence.
// Declarations, argument meaning, ownership and error behaviour: include/ahs.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cerrno>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

#include "../../include/ahs.h"
#include "features.cuh"
#include "sort.cuh"
#include "entropy.cuh"
#include "classifier.hpp"
#include "segsort.cuh"
#include "bucket.cuh"

using namespace ahs;

namespace {

// ------------------------------------------------------------ device info
struct DevInfo {
    bool ok = false;
    bool init = false;
    bool setup_failed = false;  // sm_100 device, but a kernel attribute could not be set
    int sms = 0;
    int hist_clusters = 0;  // co-resident K2 clusters
    // K6 variants: [kv][rank mode]
    // K6 variants [key width: 0 = 32-bit, 1 = 64-bit][values: 0 none, 1 32-bit, 2 64-bit][rank mode]
    const void *os_fn[2][3][2] = {};
    size_t os_smem[2][3][2] = {};
    int os_tile[2][3][2] = {};
    int os_per_sm[2][3][2] = {};  // co-resident CTAs per SM
    int os_block[2][3][2] = {};
    // 32-bit keys-only ordered passes for n >= kLargeN (sort.cuh)
    const void *osl_fn = nullptr;
    size_t osl_smem = 0;
    int osl_tile = 0, osl_per_sm = 0;
    // K6 v2 (onesweep2.cuh, hot-digit ranking) for RADIX over 32-bit keys: [0 keys, 1 pairs]
    const void *os2_fn[2] = {};
    size_t os2_smem[2] = {};
    int os2_tile[2] = {}, os2_per_sm[2] = {}, os2_block[2] = {};
    // K6 v2 10-bit pairs: key-value COUNTING with 256 < k <= 1024 in one pass (opt-in)
    const void *os10_fn = nullptr;
    size_t os10_smem = 0;
    int os10_tile = 0, os10_per_sm = 0;
    bool lane_order_ok = false;              // self-test of the ordered ranking passed
    int ent_grid[2] = {0, 0};                // K8 grid per key width (32 / 64-bit): one resident wave
    int rank_mode = kRankMasked;
};
std::mutex g_dev_mu;
DevInfo g_dev[64];

#define K2_KERNEL k_feat_hist<kHistBlock, kHistCluster>
#define K2_KERNEL64 k_feat_hist<kHistBlock, kHistCluster, uint64_t>
__device__ uint32_t g_selftest_bad;

// Runs k_lane_order_selftest on a private stream; true iff no violation.
bool lane_order_selftest(int sms)
{
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    uint32_t *bad = nullptr, zero = 0, h = 1;
    bool ok = cudaGetSymbolAddress((void **)&bad, g_selftest_bad) == cudaSuccess &&
              cudaMemcpyAsync(bad, &zero, 4, cudaMemcpyHostToDevice, st) == cudaSuccess;
    if (ok) {
        k_lane_order_selftest<<<sms, 512, 0, st>>>(bad, 288);
        ok = cudaGetLastError() == cudaSuccess &&
             cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
             cudaStreamSynchronize(st) == cudaSuccess && h == 0;
    }
    cudaGetLastError();
    cudaStreamDestroy(st);
    return ok;
}

int device_info(int *sms, int *hist_clusters = nullptr, DevInfo **info = nullptr)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return AHS_ENODEV;
    }
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevInfo &d = g_dev[dev];
    if (!d.init) {
        d.init = true;
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            cudaGetLastError();
            return AHS_ENODEV;
        }
        d.ok = (major == 10);
        if (d.ok) {
            // opt-in shared memory sizes (once per device)
            bool good = true;
            good &= cudaFuncSetAttribute(K2_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kHistSmemBytes) == cudaSuccess;
            good &= cudaFuncSetAttribute(k_feat_reduce<kReduceBlock>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kReduceSmem) == cudaSuccess;
            good &= cudaFuncSetAttribute(K2_KERNEL64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kHistSmemBytes) == cudaSuccess;
            good &= cudaFuncSetAttribute(k_feat_reduce64<kReduceBlock>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kReduceSmem) == cudaSuccess;
            if (good) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(kHistCluster * 128);
                cfg.blockDim = dim3(kHistBlock);
                cfg.dynamicSmemBytes = kHistSmemBytes;
                cudaLaunchAttribute attr;
                attr.id = cudaLaunchAttributeClusterDimension;
                attr.val.clusterDim.x = kHistCluster;
                attr.val.clusterDim.y = 1;
                attr.val.clusterDim.z = 1;
                cfg.attrs = &attr;
                cfg.numAttrs = 1;
                int nc = 0;
                if (cudaOccupancyMaxActiveClusters(&nc, (void *)K2_KERNEL, &cfg) != cudaSuccess || nc < 1) {
                    cudaGetLastError();
                    nc = d.sms / kHistCluster;
                }
                d.hist_clusters = nc;
            }
            auto set_k6 = [&](int w, int kv, int m, const void *fn, size_t smem, int tile, int block) {
                d.os_fn[w][kv][m] = fn;
                d.os_smem[w][kv][m] = smem;
                d.os_tile[w][kv][m] = tile;
                d.os_block[w][kv][m] = block;
            };
            set_k6(0, 0, kRankMasked, (const void *)K6_KEYS_M, OsKeysM::kSmem, OsKeysM::kTile, kSortBlock);
            set_k6(0, 1, kRankMasked, (const void *)K6_PAIRS_M, OsPairsM::kSmem, OsPairsM::kTile, kSortBlock);
            set_k6(0, 0, kRankOrdered, (const void *)K6_KEYS_O, OsKeysO::kSmem, OsKeysO::kTile, kSortBlock);
            set_k6(0, 1, kRankOrdered, (const void *)K6_PAIRS_O, OsPairsO::kSmem, OsPairsO::kTile, kSortBlockPairs32O);
            set_k6(1, 0, kRankMasked, (const void *)K6W_KEYS_M, OsKeys64M::kSmem, OsKeys64M::kTile, kSortBlock);
            set_k6(1, 1, kRankMasked, (const void *)K6W_PAIRS_M, OsPairs64M::kSmem, OsPairs64M::kTile, kSortBlock);
            set_k6(1, 0, kRankOrdered, (const void *)K6W_KEYS_O, OsKeys64O::kSmem, OsKeys64O::kTile,
                   kSortBlockPairsO);
            set_k6(1, 1, kRankOrdered, (const void *)K6W_PAIRS_O, OsPairs64O::kSmem, OsPairs64O::kTile,
                   kSortBlockPairsO);
            set_k6(0, 2, kRankMasked, (const void *)K6V_PAIRS_M, OsPairsV64M::kSmem, OsPairsV64M::kTile, kSortBlock);
            set_k6(0, 2, kRankOrdered, (const void *)K6V_PAIRS_O, OsPairsV64O::kSmem, OsPairsV64O::kTile,
                   kSortBlockPairsO);
            set_k6(1, 2, kRankMasked, (const void *)K6WV_PAIRS_M, OsPairs64V64M::kSmem, OsPairs64V64M::kTile, 256);
            set_k6(1, 2, kRankOrdered, (const void *)K6WV_PAIRS_O, OsPairs64V64O::kSmem, OsPairs64V64O::kTile,
                   kSortBlockPairsO);
            d.osl_fn = (const void *)K6_KEYS_OL;
            d.osl_smem = OsKeysOL::kSmem;
            d.osl_tile = OsKeysOL::kTile;
            good &= cudaFuncSetAttribute(d.osl_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.osl_smem) ==
                    cudaSuccess;
            if (good)
                good &= cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.osl_per_sm, d.osl_fn, kSortBlockOL,
                                                                      d.osl_smem) == cudaSuccess;
            good &= d.osl_per_sm > 0;
            d.os2_fn[0] = (const void *)K6V2_KEYS;
            d.os2_smem[0] = Os2Keys::kSmem;
            d.os2_tile[0] = Os2Keys::kTile;
            d.os2_block[0] = 512;
            d.os2_fn[1] = (const void *)K6V2_PAIRS;
            d.os2_smem[1] = Os2Pairs::kSmem;
            d.os2_tile[1] = Os2Pairs::kTile;
            d.os2_block[1] = kSortBlockPairsO;
            d.os10_fn = (const void *)K6V2_PAIRS10;
            d.os10_smem = Os2Pairs10::kSmem;
            d.os10_tile = Os2Pairs10::kTile;
            good &= cudaFuncSetAttribute(d.os10_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.os10_smem) ==
                    cudaSuccess;
            if (good)
                good &= cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.os10_per_sm, d.os10_fn, 256, d.os10_smem) ==
                        cudaSuccess;
            good &= d.os10_per_sm > 0;
            for (int kv = 0; kv < 2; kv++) {
                good &= cudaFuncSetAttribute(d.os2_fn[kv], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)d.os2_smem[kv]) == cudaSuccess;
                if (good)
                    good &= cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.os2_per_sm[kv], d.os2_fn[kv],
                                                                          d.os2_block[kv], d.os2_smem[kv]) ==
                            cudaSuccess;
                good &= d.os2_per_sm[kv] > 0;
            }
            for (int w = 0; w < 2; w++)
                for (int kv = 0; kv < 3; kv++)
                    for (int m = 0; m < 2; m++) {
                        // persistent K6 grids: co-resident CTAs per SM
                        good &= cudaFuncSetAttribute(d.os_fn[w][kv][m], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)d.os_smem[w][kv][m]) == cudaSuccess;
                        if (good)
                            good &= cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                        &d.os_per_sm[w][kv][m], d.os_fn[w][kv][m], d.os_block[w][kv][m],
                                        d.os_smem[w][kv][m]) == cudaSuccess;
                        good &= d.os_per_sm[w][kv][m] > 0;
                    }
            // The ordered ranking is used only if the device serves the lanes of
            // one shared atomic instruction in lane order (onesweep.cuh), checked
            // here once per device; AHS_RANK=masked forces the masked ranking.
            if (good) {
                d.lane_order_ok = lane_order_selftest(d.sms);
                const char *env = std::getenv("AHS_RANK");
                const bool force_masked = env && std::strcmp(env, "masked") == 0;
                d.rank_mode = (d.lane_order_ok && !force_masked) ? kRankOrdered : kRankMasked;
            }
            if (good) {  // K8: one wave of resident CTAs
                int per = 0;
                int per64 = 0;
                good &= cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_entropy_sorted<kEntBlock>,
                                                                      kEntBlock, 0) == cudaSuccess;
                good &= cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                            &per64, k_entropy_sorted<kEntBlock, uint64_t>, kEntBlock, 0) == cudaSuccess;
                d.ent_grid[0] = std::min(kEntMaxGrid, per * d.sms);
                d.ent_grid[1] = std::min(kEntMaxGrid, per64 * d.sms);
                good &= d.ent_grid[0] > 0 && d.ent_grid[1] > 0;
            }
            if (!good) {
                cudaGetLastError();
                d.ok = false;
                d.setup_failed = true;
            }
        }
    }
    if (!d.ok) return d.setup_failed ? AHS_ECUDA : AHS_ENODEV;
    *sms = d.sms;
    if (hist_clusters) *hist_clusters = d.hist_clusters;
    if (info) *info = &d;
    return AHS_OK;
}

// -------------------------------------------------- launch accounting / profiling
enum KernelId {
    KID_FEAT_REDUCE = 0,
    KID_FEAT_HIST,
    KID_FEAT_FINALIZE,
    KID_RADIX_HIST,
    KID_ONESWEEP,
    KID_ONESWEEP_KV,
    KID_COUNT_FILL,
    KID_COUNT_SCATTER_KV,
    KID_ENTROPY_SORTED,
    KID_HIST_SCAN,
    KID_DIGIT_COUNT,
    KID_SEG_SORT,
    KID_BUCKET_SORT,
    KID_COUNT
};
const char *kKernelNames[KID_COUNT] = {"feat_reduce", "feat_hist",   "feat_finalize",
                                       "radix_hist",  "onesweep",    "onesweep_kv",
                                       "count_fill",  "count_scatter_kv", "entropy_sorted",
                                       "hist_scan",   "digit_count64", "seg_sort", "bucket_sort"};

std::atomic<uint64_t> g_launches{0};
// NEXT-1 trivial-pass skipping (default on; AHS_SKIP_TRIVIAL=0 or ahs_set_skip_trivial(0) turn it off)
std::atomic<bool> g_skip_trivial{[] {
    const char *e = std::getenv("AHS_SKIP_TRIVIAL");
    return !(e && e[0] == '0');
}()};
// programmatic dependent launch between the kernels of a step (default on;
// AHS_PDL=0 turns it off: plain stream serialization)
std::atomic<bool> g_pdl{[] {
    const char *e = std::getenv("AHS_PDL");
    return !(e && e[0] == '0');
}()};
// key-value COUNTING with 256 < k <= 1024: one 10-bit stable scatter instead of two 8-bit radix
// passes (default off; AHS_COUNT_KV_SINGLE=1 or ahs_set_count_kv_single(1))
std::atomic<bool> g_count_kv_single{[] {
    const char *e = std::getenv("AHS_COUNT_KV_SINGLE");
    return e && e[0] == '1';
}()};
// bucket-local GENERAL plan (sort.cuh; default on where it pays: bins of >= 1536 keys on average,
// keys wider than 24 bits; AHS_BUCKET_LOCAL=0 or ahs_set_bucket_local(0) turn it off)
std::atomic<bool> g_bucket_local{[] {
    const char *e = std::getenv("AHS_BUCKET_LOCAL");
    return !(e && e[0] == '0');
}()};
// bucket-local plan with groups of several small bins per K10 segment (AHS_BL_GROUP=1; experiment)
std::atomic<bool> g_bl_group{[] {
    const char *e = std::getenv("AHS_BL_GROUP");
    return e && e[0] == '1';
}()};
// bucket-local plan: smallest mean keys per K10 segment it is chosen for (AHS_BL_MIN_KEYS; below it
// the bucket pass is no faster than the two digit passes it replaces, profiles/r02_summary.md)
const double g_bl_min_keys = [] {
    const char *e = std::getenv("AHS_BL_MIN_KEYS");
    const double v = e ? std::atof(e) : 0.0;
    return v > 0.0 ? v : 1536.0;
}();
// K10 for medium segments and the bucket pass (default on; AHS_K10=0: K9r everywhere)
std::atomic<bool> g_k10{[] {
    const char *e = std::getenv("AHS_K10");
    return !(e && e[0] == '0');
}()};
// K6 v2 for RADIX passes (default on; AHS_K6V2=0 turns it off: K6 everywhere)
std::atomic<bool> g_k6v2{[] {
    const char *e = std::getenv("AHS_K6V2");
    return !(e && e[0] == '0');
}()};
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;
struct ProfRec {
    int kid;
    cudaEvent_t a, b;
};
std::vector<ProfRec> g_prof_recs;

template <typename F>
cudaError_t launch(int kid, cudaStream_t s, F &&f)
{
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_prof.load(std::memory_order_relaxed)) {
        f();
        return cudaGetLastError();
    }
    ProfRec r{kid, nullptr, nullptr};
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, s);
    f();
    cudaError_t e = cudaGetLastError();
    cudaEventRecord(r.b, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_recs.push_back(r);
    return e;
}

// Launch a libahs kernel (every one starts with pdl_begin()) on stream s,
// with programmatic stream serialization unless AHS_PDL=0.
void pdl_config(cudaLaunchConfig_t &cfg, cudaLaunchAttribute *attr, dim3 grid, dim3 block, size_t smem,
                cudaStream_t s)
{
    cfg = cudaLaunchConfig_t{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl.load(std::memory_order_relaxed) ? 1 : 0;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args &&...args)
{
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[1];
    pdl_config(cfg, attr, grid, block, smem, s);
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------ ws layout
constexpr int kMaxReduceBlocks = 2048;
struct WsLayout {
    size_t feat, partials, fctrl, ovf, hist, scan, parts, byte0, digit1, ent, total;
};
WsLayout ws_layout()
{
    WsLayout L;
    size_t o = 0;
    L.feat = o;
    o += align_up(sizeof(DevFeatures), 256);
    L.partials = o;
    o += align_up(sizeof(Partial64) * kMaxReduceBlocks, 256);  // 32- or 64-bit partials
    L.fctrl = o;
    o += align_up(sizeof(FinalCtrl), 256);
    L.ovf = o;
    o += (size_t)kMaxBins * 4;
    L.hist = o;
    o += (size_t)kMaxBins * 4;
    L.scan = o;
    o += align_up((size_t)(kMaxBins + 1) * 4, 256);
    L.parts = o;
    o += (size_t)kMaxHistRows * kMaxBins * 4;
    L.byte0 = o;  // K1: per-CTA histograms of the raw low byte (radix digit 0)
    o += (size_t)kMaxReduceBlocks * 256 * 4;
    L.digit1 = o;  // K2: per-CTA histograms of digit 1 of key - min (when shift > 8)
    o += (size_t)kMaxHistRows * kHistCluster * 256 * 4;
    L.ent = o;  // K8 (NEXT-2): per-chunk run pieces, per-chunk sums, result
    o += align_up((size_t)kEntMaxGrid * (sizeof(RunPieces) + 8) + 256, 256);
    L.total = o;
    return L;
}

// ------------------------------------------------------------ tmp layout
// [ctrl: digit histograms, bucket bases (kMaxPasses x 256 u32 each), 256 B of
//  tickets (passes 0..7, K5 at [8]) and the pass plan (at [16], kMaxPasses + 2
//  words)] [look-back status: room for two regions at the smallest K6 tile;
//  a sort uses two regions of its own tile count, back to back, alternating
//  between passes] [second key buffer (n x key bytes)] [second value buffer]
// The ctrl block sits at offset 0 whatever n and the key width.
struct TmpLayout {
    size_t ctrl, dhist, bucket, ticket, status, status_region_bytes, keys, vals, total;
};
constexpr int kTicketPlan = 16;   // plan offset in the ticket block (words)
constexpr int kTicketFault = 32;  // K6 look-back gave up (onesweep.cuh kLookbackSpinLimit): AHS_ECUDA
constexpr int kTicketMaxBin = kMaxPasses + 1;  // K5: largest feature-bin count (bucket-local plan)
constexpr int kTicketSegBad = 33;              // K10: buckets above the segment sort's capacity (never, by K5)
TmpLayout tmp_layout(uint64_t n, int has_vals, size_t key_bytes = 4, size_t val_bytes = 4)
{
    TmpLayout L;
    size_t o = 0;
    L.ctrl = o;
    L.dhist = o;
    L.bucket = o + (size_t)kMaxPasses * 256 * 4;
    L.ticket = o + 2 * (size_t)kMaxPasses * 256 * 4;
    o += 2 * (size_t)kMaxPasses * 256 * 4 + 256;
    L.status = o;
    const uint64_t tiles = (n + kMinTile - 1) / kMinTile;
    L.status_region_bytes = align_up((size_t)tiles * kBins * 4, 256);
    if (has_vals && key_bytes == 4 && val_bytes == 4) {
        // the single 10-bit COUNTING scatter (Os2Pairs10) uses both regions as one: 1024 statuses per tile
        const uint64_t t10 = (n + Os2Pairs10::kTile - 1) / Os2Pairs10::kTile;
        L.status_region_bytes = std::max(L.status_region_bytes, align_up((size_t)t10 * 1024 * 4 / 2 + 256, 256));
    }
    o += 2 * L.status_region_bytes;
    L.keys = o;
    o += align_up(n * key_bytes, 256);
    L.vals = o;
    if (has_vals) o += align_up(n * val_bytes, 256);
    L.total = o;
    return L;
}

inline bool dtype_valid(int32_t dtype)
{
    return dtype == AHS_I32 || dtype == AHS_U32 || dtype == AHS_I64 || dtype == AHS_U64;
}
inline bool dtype_wide(int32_t dtype) { return dtype == AHS_I64 || dtype == AHS_U64; }
inline size_t key_bytes_of(int32_t dtype) { return dtype_wide(dtype) ? 8 : 4; }
inline uint32_t flip_of(int32_t dtype) { return dtype == AHS_I32 ? 0x80000000u : 0u; }
inline uint64_t flip64_of(int32_t dtype) { return dtype == AHS_I64 ? 0x8000000000000000ull : 0ull; }
inline uint32_t umin_of(const ahs_features_t *f) { return (uint32_t)f->min ^ flip_of((int32_t)f->dtype); }
inline uint64_t umin64_of(const ahs_features_t *f) { return (uint64_t)f->min ^ flip64_of((int32_t)f->dtype); }

bool thresholds_valid(const ahs_thresholds_t *th)
{
    return th->n_insertion > 0 && th->k_counting > 0 && th->k_radix > 0 &&
           th->k_counting < th->k_radix && th->entropy_coeff > 0.0 && th->entropy_coeff <= 1.0 &&
           (th->entropy_norm == AHS_NORM_BUCKETS || th->entropy_norm == AHS_NORM_RANGE) &&
           th->reserved == 0;
}

int radix_passes(uint32_t bits) { return (int)((bits + 7u) / 8u); }





}  // namespace

// ====================================================================== API
extern "C" {

const char *ahs_version(void) { return "ahs-b200 0.1 (sm_100a)"; }

const char *ahs_status_string(int s)
{
    switch (s) {
    case AHS_OK: return "ok";
    case AHS_EINVAL: return "invalid argument";
    case AHS_ENOSPACE: return "workspace or tmp buffer too small";
    case AHS_ERANGE: return "n exceeds AHS_MAX_N";
    case AHS_EFEAT: return "features do not match the keys (n or dtype)";
    case AHS_ECUDA: return "CUDA error";
    case AHS_ENODEV: return "no sm_100 CUDA device";
    case AHS_EMODEL: return "malformed or invalid model";
    case AHS_EMODELVER: return "unsupported model version";
    default: return "unknown status";
    }
}

void ahs_thresholds_default(ahs_thresholds_t *th)
{
    if (!th) return;
    th->n_insertion = 20;      // Table II
    th->k_counting = 1024;     // Table II
    th->k_radix = 1000000;     // Table II
    th->entropy_coeff = 0.7;
    th->entropy_norm = AHS_NORM_BUCKETS;
    th->reserved = 0;
}

// SURVEY §5 Config/flags: environment overrides of the Table II thresholds, named after SPEC's CLI
// flags.  Malformed or invalid values -> AHS_EINVAL (th keeps the defaults).
int ahs_thresholds_from_env(ahs_thresholds_t *th)
{
    if (!th) return AHS_EINVAL;
    ahs_thresholds_t t;
    ahs_thresholds_default(&t);
    auto u64 = [](const char *name, uint64_t *out) -> bool {
        const char *e = std::getenv(name);
        if (!e || !*e) return true;
        char *end = nullptr;
        errno = 0;
        const unsigned long long v = std::strtoull(e, &end, 10);
        if (errno || !end || *end || e[0] == '-') return false;
        *out = (uint64_t)v;
        return true;
    };
    bool ok = u64("AHS_N_INSERTION", &t.n_insertion) && u64("AHS_K_COUNTING", &t.k_counting) &&
              u64("AHS_K_RADIX", &t.k_radix);
    if (const char *e = std::getenv("AHS_ENTROPY_COEFF"); ok && e && *e) {
        char *end = nullptr;
        errno = 0;
        t.entropy_coeff = std::strtod(e, &end);
        ok = !errno && end && !*end;
    }
    if (const char *e = std::getenv("AHS_ENTROPY_NORM"); ok && e && *e) {
        if (!std::strcmp(e, "buckets") || !std::strcmp(e, "0")) t.entropy_norm = AHS_NORM_BUCKETS;
        else if (!std::strcmp(e, "range") || !std::strcmp(e, "1")) t.entropy_norm = AHS_NORM_RANGE;
        else ok = false;
    }
    ahs_thresholds_default(th);
    if (!ok || !thresholds_valid(&t)) return AHS_EINVAL;
    *th = t;
    return AHS_OK;
}

size_t ahs_workspace_bytes(uint64_t) { return ws_layout().total; }

size_t ahs_sort_tmp_bytes(uint64_t n, int has_vals) { return tmp_layout(n, has_vals).total; }

size_t ahs_sort_tmp_bytes_dtype(uint64_t n, int has_vals, int32_t dtype)
{
    return dtype_valid(dtype) ? tmp_layout(n, has_vals, key_bytes_of(dtype)).total : 0;
}

size_t ahs_sort_tmp_bytes_ex(uint64_t n, uint32_t value_bytes, int32_t dtype)
{
    if (!dtype_valid(dtype) || (value_bytes != 0 && value_bytes != 4 && value_bytes != 8)) return 0;
    return tmp_layout(n, value_bytes != 0, key_bytes_of(dtype), value_bytes ? value_bytes : 4).total;
}

int ahs_sort_passes(const ahs_features_t *f, int32_t strategy, int has_vals)
{
    if (!f) return AHS_EINVAL;
    if (f->n == 0 || f->k <= 1) return 0;
    switch (strategy) {
    case AHS_GENERAL: return dtype_wide((int32_t)f->dtype) ? 8 : 4;
    case AHS_RADIX: return radix_passes(f->bits);
    case AHS_COUNTING:
        if (f->shift > 0) return radix_passes(f->bits);
        if (!has_vals) return 0;
        if (f->bits <= 8) return 1;
        if (f->bits <= 10 && !dtype_wide((int32_t)f->dtype) && g_count_kv_single.load()) {
            int sms = 0;
            DevInfo *di = nullptr;
            if (device_info(&sms, nullptr, &di) == AHS_OK && di->rank_mode == kRankOrdered) return 1;
        }
        return radix_passes(f->bits);
    default: return AHS_EINVAL;
    }
}

uint64_t ahs_launch_count(void) { return g_launches.load(); }

int ahs_rank_mode(int mode)
{
    int sms = 0;
    DevInfo *di = nullptr;
    int rc = device_info(&sms, nullptr, &di);
    if (rc) return rc;
    if (mode == -1) return di->rank_mode;
    if (mode == AHS_RANK_MASKED) {
        di->rank_mode = kRankMasked;
    } else if (mode == AHS_RANK_ORDERED) {
        if (!di->lane_order_ok) return AHS_EINVAL;
        di->rank_mode = kRankOrdered;
    } else {
        return AHS_EINVAL;
    }
    return di->rank_mode;
}

int ahs_set_skip_trivial(int on)
{
    if (on != 0 && on != 1) return g_skip_trivial.load() ? 1 : 0;
    g_skip_trivial.store(on == 1);
    return on;
}

int ahs_set_count_kv_single(int on)
{
    if (on != 0 && on != 1) return g_count_kv_single.load() ? 1 : 0;
    g_count_kv_single.store(on == 1);
    return on;
}

// the plan block of the last ahs_sort on d_tmp (synchronizes): executed digit passes, bucket-local
// flag; AHS_ECUDA when a look-back gave up; -1 passes when that sort wrote no plan
static int read_plan(const void *d_tmp, size_t tmp_bytes, int *passes, int *bl, void *stream)
{
    const TmpLayout TL = tmp_layout(0, 0);  // the ctrl block does not depend on n or the key width
    if (!d_tmp || tmp_bytes < TL.status) return AHS_EINVAL;
    uint32_t w[kPlanBL + 1];
    uint32_t fault = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemcpyAsync(w, (const char *)d_tmp + TL.ticket + kTicketPlan * 4, sizeof(w), cudaMemcpyDeviceToHost,
                        s) != cudaSuccess ||
        cudaMemcpyAsync(&fault, (const char *)d_tmp + TL.ticket + kTicketFault * 4, 4, cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        cudaGetLastError();
        return AHS_ECUDA;
    }
    if (fault) return AHS_ECUDA;
    const bool has = w[kMaxPasses + 1] == kPlanMagic;
    *passes = has ? (int)w[kMaxPasses] : -1;
    *bl = has && w[kPlanBL] ? 1 : 0;
    return AHS_OK;
}

int ahs_sort_executed_passes(const void *d_tmp, size_t tmp_bytes, uint64_t n, int has_vals, void *stream)
{
    (void)n;
    (void)has_vals;
    int p = -1, bl = 0;
    const int rc = read_plan(d_tmp, tmp_bytes, &p, &bl, stream);
    if (rc) return rc;
    return p < 0 ? p : p + bl;  // the bucket-local pass reads and writes every key once, like a digit pass
}

int ahs_sort_plan(const void *d_tmp, size_t tmp_bytes, int *digit_passes, int *bucket_local, void *stream)
{
    if (!digit_passes || !bucket_local) return AHS_EINVAL;
    return read_plan(d_tmp, tmp_bytes, digit_passes, bucket_local, stream);
}

int ahs_set_bucket_local(int on)
{
    if (on != 0 && on != 1) return g_bucket_local.load() ? 1 : 0;
    g_bucket_local.store(on == 1);
    return on;
}

int ahs_lane_order_ok(void)
{
    int sms = 0;
    DevInfo *di = nullptr;
    int rc = device_info(&sms, nullptr, &di);
    if (rc) return rc;
    return di->lane_order_ok ? 1 : 0;
}
int ahs_kernel_count(void) { return KID_COUNT; }
const char *ahs_kernel_name(int id) { return (id >= 0 && id < KID_COUNT) ? kKernelNames[id] : ""; }

int ahs_profile_begin(void)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof_recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof_recs.clear();
    g_prof.store(true);
    return AHS_OK;
}

int ahs_profile_end(void)
{
    g_prof.store(false);
    return AHS_OK;
}

int ahs_profile_read(double *ms, uint64_t *launches, int n_ids)
{
    if (!ms || !launches || n_ids < KID_COUNT) return AHS_EINVAL;
    for (int i = 0; i < n_ids; i++) {
        ms[i] = 0.0;
        launches[i] = 0;
    }
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof_recs) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) return AHS_ECUDA;
        float t = 0.f;
        if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return AHS_ECUDA;
        ms[r.kid] += t;
        launches[r.kid] += 1;
    }
    return AHS_OK;
}

// --------------------------------------------------------------- features
int ahs_features(const void *d_keys, uint64_t n, int32_t dtype, void *d_ws, size_t ws_bytes,
                 ahs_features_t *feat, void *stream)
{
    if (!feat || !dtype_valid(dtype)) return AHS_EINVAL;
    std::memset(feat, 0, sizeof(*feat));
    feat->n = n;
    feat->dtype = (uint32_t)dtype;
    feat->entropy_bits = AHS_ENTROPY_BITS;
    if (dtype == AHS_I32 || dtype == AHS_I64) feat->flags |= AHS_FLAG_SIGNED;
    const bool wide = dtype_wide(dtype);
    if (n == 0) {  // empty input exits in O(1)
        feat->flags |= AHS_FLAG_EMPTY | AHS_FLAG_SORTED;
        return AHS_OK;
    }
    if (n > AHS_MAX_N) return AHS_ERANGE;
    if (!d_keys || !d_ws || ((uintptr_t)d_keys & (key_bytes_of(dtype) - 1)) || ((uintptr_t)d_ws & 15u))
        return AHS_EINVAL;
    const WsLayout L = ws_layout();
    if (ws_bytes < L.total) return AHS_ENOSPACE;
    int sms = 0, hclusters = 0;
    int rc = device_info(&sms, &hclusters);
    if (rc) return rc;

    cudaStream_t s = (cudaStream_t)stream;
    char *ws = (char *)d_ws;
    const uint32_t *keys = (const uint32_t *)d_keys;
    const uint32_t flip = flip_of(dtype);
    Partial *partials = (Partial *)(ws + L.partials);
    FinalCtrl *fctrl = (FinalCtrl *)(ws + L.fctrl);
    uint32_t *ovf = (uint32_t *)(ws + L.ovf);
    uint32_t *hist = (uint32_t *)(ws + L.hist);
    uint32_t *parts = (uint32_t *)(ws + L.parts);
    DevFeatures *dfeat = (DevFeatures *)(ws + L.feat);

    const uint64_t nvec = wide ? n / 2 : n / 4;  // 16-byte vectors
    const uint64_t nch1 = (nvec + kReduceChunk / 16 - 1) / (kReduceChunk / 16);
    const uint64_t g1 = std::max<uint64_t>(1, std::min<uint64_t>(nch1, (uint64_t)sms * 2));
    const uint64_t *keys64 = (const uint64_t *)d_keys;
    Partial64 *partials64 = (Partial64 *)(ws + L.partials);
    const uint64_t flip64 = flip64_of(dtype);

    cudaError_t e = launch(KID_FEAT_REDUCE, s, [&] {
        if (wide)
            launch_k(k_feat_reduce64<kReduceBlock>, dim3((unsigned)g1), dim3(kReduceBlock), kReduceSmem, s, keys64,
                     n, flip64, partials64, ovf, kMaxBins, fctrl, (uint32_t *)(ws + L.byte0));
        else
            launch_k(k_feat_reduce<kReduceBlock>, dim3((unsigned)g1), dim3(kReduceBlock), kReduceSmem, s, keys, n,
                     flip, partials, ovf, kMaxBins, fctrl, (uint32_t *)(ws + L.byte0));
    });
    if (e != cudaSuccess) return AHS_ECUDA;
    // K2: clusters of kHistCluster CTAs, one partial-histogram row per cluster
    const uint64_t nch2 = (nvec + kHistChunk / 16 - 1) / (kHistChunk / 16);
    uint64_t rows = (nch2 + kHistCluster - 1) / kHistCluster;
    rows = std::max<uint64_t>(1, std::min<uint64_t>(rows, (uint64_t)std::min(hclusters, kMaxHistRows)));
    e = launch(KID_FEAT_HIST, s, [&] {
        if (wide)
            launch_k(K2_KERNEL64, dim3((unsigned)(rows * kHistCluster)), dim3(kHistBlock), kHistSmemBytes, s, keys64,
                     n, flip64, (const Partial64 *)partials64, (int)g1, ovf, parts, (uint32_t *)(ws + L.digit1), fctrl);
        else
            launch_k(K2_KERNEL, dim3((unsigned)(rows * kHistCluster)), dim3(kHistBlock), kHistSmemBytes, s, keys, n,
                     flip, (const Partial *)partials, (int)g1, ovf, parts, (uint32_t *)(ws + L.digit1), fctrl);
    });
    if (e != cudaSuccess) return AHS_ECUDA;
    // the one host sync of the pipeline: K3's last CTA writes the 64-byte
    // feature record straight into a per-thread mapped pinned buffer and
    // releases its sequence word; the host polls that word (no copy, no
    // stream sync).  Without a mapped buffer: copy + stream sync.
    struct HostFeat {
        DevFeatures *h = nullptr, *d = nullptr;
        uint64_t seq = 0;
        bool tried = false;
    };
    thread_local HostFeat hfb;
    if (!hfb.tried) {
        hfb.tried = true;
        if (cudaHostAlloc((void **)&hfb.h, sizeof(DevFeatures), cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer((void **)&hfb.d, hfb.h, 0) != cudaSuccess) {
            cudaGetLastError();
            if (hfb.h) cudaFreeHost(hfb.h);
            hfb.h = hfb.d = nullptr;
        } else {
            std::memset(hfb.h, 0, sizeof(DevFeatures));
        }
    }
    const uint64_t seq = ++hfb.seq;
    e = launch(KID_FEAT_FINALIZE, s, [&] {
        if (wide)
            launch_k(k_feat_finalize<kFinalBlock, kFinalGroups, uint64_t>, dim3(kFinalGrid), dim3(kFinalBlock), 0,
                     s, n, (int)g1, (const uint32_t *)parts, (int)rows,
                     (const uint32_t *)ovf, hist, fctrl, dfeat, hfb.d, seq);
        else
            launch_k(k_feat_finalize<kFinalBlock, kFinalGroups>, dim3(kFinalGrid), dim3(kFinalBlock), 0, s, n,
                     (int)g1, (const uint32_t *)parts, (int)rows, (const uint32_t *)ovf,
                     hist, fctrl, dfeat, hfb.d, seq);
    });
    if (e != cudaSuccess) return AHS_ECUDA;

    DevFeatures hf;
    if (hfb.h) {
        volatile uint64_t *flag = &hfb.h->seq;
        // spin while the record is close (the device-resident case: tens of us); once
        // the wait is long (an upload ahead of it on the stream), yield between polls
        // so concurrent callers' threads are not starved of cores
        const auto t0 = std::chrono::steady_clock::now();
        bool polite = false;
        for (uint32_t spin = 0;; spin++) {
            if (*flag == seq) break;
            if (polite) std::this_thread::yield();
            if ((spin & 255u) == 255u) {  // the kernel may have failed: stream state
                if (!polite && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(100)) polite = true;
                const cudaError_t q = cudaStreamQuery(s);
                if (q == cudaSuccess) {
                    if (*flag == seq) break;
                    return AHS_ECUDA;  // stream drained without the record
                }
                if (q != cudaErrorNotReady) {
                    cudaGetLastError();
                    return AHS_ECUDA;
                }
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        std::memcpy(&hf, (const void *)hfb.h, sizeof(hf));
    } else {
        if (cudaMemcpyAsync(&hf, dfeat, sizeof(hf), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            cudaGetLastError();
            return AHS_ECUDA;
        }
    }
    // min / max from the ordered images: the key's value (uint64: its bit pattern)
    switch (dtype) {
    case AHS_I32:
        feat->min = (int64_t)(int32_t)((uint32_t)hf.umin ^ 0x80000000u);
        feat->max = (int64_t)(int32_t)((uint32_t)hf.umax ^ 0x80000000u);
        break;
    case AHS_I64:
        feat->min = (int64_t)(hf.umin ^ 0x8000000000000000ull);
        feat->max = (int64_t)(hf.umax ^ 0x8000000000000000ull);
        break;
    default:
        feat->min = (int64_t)hf.umin;
        feat->max = (int64_t)hf.umax;
        break;
    }
    if (hf.ksat) feat->flags |= AHS_FLAG_K_SATURATED;
    feat->k = hf.k;
    feat->bits = hf.bits;
    feat->shift = hf.shift;
    feat->nbins = hf.nb;
    feat->entropy = hf.entropy;
    feat->descents = hf.descents;
    if (hf.k == 1) feat->flags |= AHS_FLAG_CONSTANT;
    if (hf.shift > 0) feat->flags |= AHS_FLAG_BUCKETED;
    if (hf.descents == 0) feat->flags |= AHS_FLAG_SORTED;
    if (n >= 2 && hf.descents == n - 1) feat->flags |= AHS_FLAG_STRICT_DESC;
    return AHS_OK;
}

// K3s: the exclusive scan of the feature histogram (COUNTING only); returns
// the device scan array in ws, or nullptr on a launch error.
static const uint32_t *hist_scan(void *d_ws, const ahs_features_t *feat, cudaStream_t s)
{
    const WsLayout L = ws_layout();
    char *ws = (char *)d_ws;
    uint32_t *scan = (uint32_t *)(ws + L.scan);
    const unsigned g = (unsigned)((feat->nbins + kScanBlock - 1) / kScanBlock);
    const cudaError_t e = launch(KID_HIST_SCAN, s, [&] {
        launch_k(k_hist_scan<kScanBlock>, dim3(g), dim3(kScanBlock), 0, s, (const uint32_t *)(ws + L.hist),
                 (const FinalCtrl *)(ws + L.fctrl), feat->nbins, (uint32_t)feat->n, scan);
    });
    return e == cudaSuccess ? scan : nullptr;
}

// ----------------------------------------------------------------- select
int ahs_select(const ahs_features_t *f, const ahs_thresholds_t *th, int32_t *strategy, int32_t *rule)
{
    ahs_thresholds_t def;
    if (!th) {
        ahs_thresholds_default(&def);
        th = &def;
    }
    if (!f || !strategy || !thresholds_valid(th)) return AHS_EINVAL;
    int32_t st, ru;
    if (f->n == 0) {                       // P:411 empty
        st = AHS_COUNTING;
        ru = AHS_RULE_EMPTY;
    } else if (f->k == 1) {                // P:411 constant (k = 1)
        st = AHS_COUNTING;
        ru = AHS_RULE_CONSTANT;
    } else if (f->n <= th->n_insertion) {  // P:96 n <= 20 -> Insertion
        st = AHS_GENERAL;
        ru = AHS_RULE_SMALL_N;
    } else if (f->k <= th->k_counting) {   // P:96 k <= 1000 (Table II: 1,024) -> Counting
        st = AHS_COUNTING;
        ru = AHS_RULE_SMALL_RANGE;
    } else if (f->k > th->k_radix &&       // P:98 k > 10^6 and H < 0.7 log2 k -> Radix
               f->entropy < th->entropy_coeff *
                                std::log2(th->entropy_norm == AHS_NORM_RANGE ? (double)f->k
                                                                              : (double)f->nbins)) {
        st = AHS_RADIX;
        ru = AHS_RULE_LOW_ENTROPY;
    } else {                               // P:98 otherwise QuickSort
        st = AHS_GENERAL;
        ru = AHS_RULE_DEFAULT;
    }
    *strategy = st;
    if (rule) *rule = ru;
    return AHS_OK;
}

// ------------------------------------------------------------------- sort
}  // extern "C"

namespace {
// The digit passes of ahs_sort for key type K (uint32_t, or uint64_t: NEXT-3).
// the K9 segment sort launcher (defined with ahs_sort_segments below), used by the bucket-local plan
template <typename K, bool KV>
cudaError_t seg_launch(const void *kin, const uint32_t *vin, void *kout, uint32_t *vout, uint64_t n,
                       const uint32_t *offsets, uint32_t nseg, uint32_t max_segment, K flip, uint32_t *bad,
                       bool ord, cudaStream_t s, const uint32_t *gate = nullptr, uint32_t group = 1, K sub = 0);

template <typename K, typename V>
int sort_impl(const K *kin, const V *d_vals_in, K *kout, V *d_vals_out, uint64_t n, int32_t strategy,
              const ahs_features_t *feat, void *d_ws, size_t ws_bytes, void *d_tmp, size_t tmp_bytes,
              cudaStream_t s)
{
    constexpr bool kWide = sizeof(K) == 8;
    constexpr int W = kWide ? 1 : 0;
    const int32_t dtype = (int32_t)feat->dtype;
    const bool kv = d_vals_in != nullptr;
    const int VK = kv ? (sizeof(V) == 8 ? 2 : 1) : 0;  // K6 variant: no values / 32-bit / 64-bit
    int sms = 0;
    DevInfo *di = nullptr;
    int rc = device_info(&sms, nullptr, &di);
    if (rc) return rc;
    const K flip = kWide ? (K)flip64_of(dtype) : (K)flip_of(dtype);
    const K umin = kWide ? (K)umin64_of(feat) : (K)umin_of(feat);
    const uint32_t n32 = (uint32_t)n;

    // paths without digit passes still clear the plan and look-back fault words of a reused d_tmp
    // (ticket words kTicketPlan .. kTicketFault; the digit-pass path clears the whole control block)
    auto clear_fault = [&]() -> bool {
        const TmpLayout T0 = tmp_layout(0, 0);
        if (!d_tmp || tmp_bytes < T0.status) return true;
        return cudaMemsetAsync((char *)d_tmp + T0.ticket + kTicketPlan * 4, 0, (kTicketFault - kTicketPlan + 1) * 4,
                               s) == cudaSuccess;
    };
    // constant input: stable identity
    if (feat->k == 1) {
        if (!clear_fault()) return AHS_ECUDA;
        if (kout != kin && cudaMemcpyAsync(kout, kin, n * sizeof(K), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return AHS_ECUDA;
        if (kv && d_vals_out != d_vals_in &&
            cudaMemcpyAsync(d_vals_out, d_vals_in, n * sizeof(V), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return AHS_ECUDA;
        return AHS_OK;
    }

    const WsLayout WL = ws_layout();
    const bool exact_hist = feat->shift == 0 && feat->nbins == feat->k;
    // ---- keys-only COUNTING from the feature histogram (Listing 2)
    if (strategy == AHS_COUNTING && exact_hist && !kv) {
        if (!d_ws || ws_bytes < WL.total) return AHS_ENOSPACE;
        if (!clear_fault()) return AHS_ECUDA;
        const uint32_t *scan = hist_scan(d_ws, feat, s);
        if (!scan) return AHS_ECUDA;
        cudaError_t e;
        if constexpr (kWide) {
            const uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>((n + kFill64Block - 1) / kFill64Block,
                                                                        (uint64_t)sms * 8));
            e = launch(KID_COUNT_FILL, s, [&] {
                launch_k(k_count_fill64, dim3((unsigned)g), dim3(kFill64Block), 0, s, kout, n32, scan, feat->nbins,
                         flip, umin);
            });
        } else {
            const uint64_t nvec = n / 4;
            uint64_t g = (4 * nvec + kFillChunk - 1) / kFillChunk;
            g = std::max<uint64_t>(1, g);
            e = launch(KID_COUNT_FILL, s, [&] {
                launch_k(k_count_fill, dim3((unsigned)g), dim3(kFillBlock), 0, s, kout, n32, scan, feat->nbins, flip,
                         umin);
            });
        }
        return e == cudaSuccess ? AHS_OK : AHS_ECUDA;
    }

    // ---- digit passes: plan
    const TmpLayout TL = tmp_layout(n, kv, sizeof(K), sizeof(V));
    if (!d_tmp || tmp_bytes < TL.total || ((uintptr_t)d_tmp & 255u)) return AHS_ENOSPACE;
    char *tmp = (char *)d_tmp;
    K *tkeys = (K *)(tmp + TL.keys);
    V *tvals = kv ? (V *)(tmp + TL.vals) : nullptr;
    uint32_t *dhist = (uint32_t *)(tmp + TL.dhist);
    uint32_t *bucket = (uint32_t *)(tmp + TL.bucket);
    uint32_t *tickets = (uint32_t *)(tmp + TL.ticket);
    uint32_t *status = (uint32_t *)(tmp + TL.status);

    const bool count_kv8 = strategy == AHS_COUNTING && exact_hist && kv && feat->bits <= 8;
    const bool count_kv10 = strategy == AHS_COUNTING && exact_hist && kv && feat->bits > 8 && feat->bits <= 10 &&
                            W == 0 && VK == 1 && di->rank_mode == kRankOrdered && g_count_kv_single.load();
    const bool count_kv = count_kv8 || count_kv10;  // one stable scatter by key - min (Listing 2)
    int passes;
    if (count_kv) passes = 1;
    else if (strategy == AHS_GENERAL) passes = kWide ? 8 : 4;  // full width, on key - min (R14)
    else passes = radix_passes(feat->bits);                     // RADIX, or COUNTING without the histogram

    // passes alternate between two status regions; the host zeroes the control words and the first
    // pass's region (one memset), and each pass clears the other region at its end for the next
    const int mode = di->rank_mode;
    // RADIX over 32-bit keys (ordered ranking): K6 v2 with the hot-digit ranking (low-entropy
    // inputs have skewed digits); everything else: K6
    const bool v2 = W == 0 && VK < 2 && mode == kRankOrdered && strategy == AHS_RADIX && !count_kv &&
                    g_k6v2.load(std::memory_order_relaxed);
    const bool large = !v2 && W == 0 && VK == 0 && mode == kRankOrdered && n >= kLargeN;
    const uint64_t tile = v2 ? (uint64_t)di->os2_tile[VK]
                        : large ? (uint64_t)di->osl_tile : (uint64_t)di->os_tile[W][VK][mode];
    const uint64_t tiles = (n + tile - 1) / tile;
    const int per_sm = v2 ? di->os2_per_sm[VK] : large ? di->osl_per_sm : di->os_per_sm[W][VK][mode];
    const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)sms * per_sm);
    const void *k6 = v2 ? di->os2_fn[VK] : large ? di->osl_fn : di->os_fn[W][VK][mode];
    size_t k6_smem = v2 ? di->os2_smem[VK] : large ? di->osl_smem : di->os_smem[W][VK][mode];
    unsigned k6_block = v2 ? (unsigned)di->os2_block[VK]
                      : large ? (unsigned)kSortBlockOL : (unsigned)di->os_block[W][VK][mode];
    unsigned grid_k6 = grid;
    if (count_kv10) {
        k6 = di->os10_fn;
        k6_smem = di->os10_smem;
        k6_block = 256;
        const uint64_t t10 = (n + di->os10_tile - 1) / di->os10_tile;
        grid_k6 = (unsigned)std::min<uint64_t>(t10, (uint64_t)sms * di->os10_per_sm);
    }
    // statuses of one pass; the 10-bit COUNTING scatter (1024 per tile) spans both regions
    const size_t status_words_per_pass =
        count_kv10 ? (size_t)((n + di->os10_tile - 1) / di->os10_tile) * 1024 : (size_t)tiles * kBins;
    // the control words and the first pass's status region; each pass clears the other region for
    // the next one at its end (pass 0: region 1, still dirty)
    const size_t zero_bytes = (TL.status - TL.ctrl) + status_words_per_pass * 4;
    if (cudaMemsetAsync(tmp + TL.ctrl, 0, zero_bytes, s) != cudaSuccess) return AHS_ECUDA;

    // in place with an odd pass count: stream the input to tmp first.  In place,
    // the pass count (and so the buffer parity) must be known here: no skipping.
    const K *src_k = kin;
    const V *src_v = d_vals_in;
    const bool inplace = kout == kin || (kv && d_vals_out == d_vals_in);
    const bool skip = !inplace && g_skip_trivial.load() && !count_kv;
    if (inplace && (passes & 1)) {
        if (cudaMemcpyAsync(tkeys, kin, n * sizeof(K), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return AHS_ECUDA;
        if (kv && cudaMemcpyAsync(tvals, d_vals_in, n * sizeof(V), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return AHS_ECUDA;
        src_k = tkeys;
        src_v = tvals;
    }

    if (!d_ws || ws_bytes < WL.total) return AHS_ENOSPACE;
    uint32_t *plan = tickets + kTicketPlan;
    // bucket-local plan candidate (GENERAL over 32-bit keys with <= 32-bit values, buckets of the
    // feature histogram coarser than single values): two passes over the bin digits + K10.  K5 takes
    // it when the largest bin fits the K10 capacity chosen here from the mean bin size.
    uint32_t bl_cap = 0, bl_group = 1;
    const uint32_t *bl_offsets = nullptr;
    if (strategy == AHS_GENERAL && W == 0 && VK <= 1 && !inplace && feat->shift > 0 && passes == 4 &&
        g_bucket_local.load(std::memory_order_relaxed)) {
        // K10 sorts groups of G consecutive bins as one segment (the array is ordered by bin after the
        // two bin-digit passes): G doubles while a group stays <= ~4096 keys and its bin bits stay inside
        // the digits the low s bits already use (no extra sub-pass).  Capacity: the group mean plus six
        // standard deviations of a uniform fill.  Below ~1500 keys per group the bucket pass is no
        // faster than the two digit passes it replaces (profiles/r02_summary.md).
        const double mean = (double)n / (double)feat->nbins;
        const uint32_t low_digits = (feat->shift + 7u) / 8u;
        while (g_bl_group.load(std::memory_order_relaxed) && mean * 2.0 * bl_group <= 4096.0 &&
               feat->shift + (uint32_t)__builtin_ctz(bl_group * 2u) <= 8u * low_digits)
            bl_group *= 2u;
        const double gm = mean * bl_group;
        const double need = gm + 6.0 * std::sqrt(gm) + 32.0;
        if (gm >= g_bl_min_keys)
            for (uint32_t c : {1536u, 2048u, 4096u, 4608u, 5120u, 6144u, 8192u})
                if (need <= (double)c) {
                    bl_cap = c;
                    break;
                }
        if (bl_cap) {
            bl_offsets = hist_scan(d_ws, feat, s);  // bucket boundaries: scan[b] .. scan[b + 1]
            if (!bl_offsets) return AHS_ECUDA;
        }
    }
    const uint32_t *bases;
    if (count_kv) {
        bases = hist_scan(d_ws, feat, s);
        if (!bases) return AHS_ECUDA;
    } else {
        const char *wsc = (const char *)d_ws;
        const uint32_t *fhist = (const uint32_t *)(wsc + WL.hist);
        cudaError_t e = cudaSuccess;
        if constexpr (kWide) {
            // K5b: digits 2 .. below the feature buckets come from the keys
            const int p1 = std::min(passes, (int)((feat->shift + 7) / 8));
            if (p1 > 2) {
                const uint64_t g = std::max<uint64_t>(
                    1, std::min<uint64_t>((n + kDC64Block - 1) / kDC64Block, (uint64_t)sms * 4));
                e = launch(KID_DIGIT_COUNT, s, [&] {
                    launch_k(k_digit_count64<kDC64Block>, dim3((unsigned)g), dim3(kDC64Block), 0, s,
                             (const uint64_t *)src_k, n, (uint64_t)(umin - flip), 2, p1, dhist);
                });
                if (e != cudaSuccess) return AHS_ECUDA;
            }
        }
        const uint64_t g5 = std::max<uint64_t>(2 * kRowCtas, ((uint64_t)feat->nbins + kRHBlock - 1) / kRHBlock);
        e = launch(KID_RADIX_HIST, s, [&] {
            launch_k(k_radix_hist<kRHBlock, kWide ? 8 : 4>, dim3((unsigned)g5), dim3(kRHBlock), 0, s, n,
                     (uint32_t)umin, passes, fhist, feat->nbins, feat->shift, (const DevFeatures *)(wsc + WL.feat),
                     (const uint32_t *)(wsc + WL.byte0), (const uint32_t *)(wsc + WL.digit1), dhist, bucket,
                     tickets + kMaxPasses, plan, skip ? 1 : 0, bl_cap, bl_group, tickets + kTicketMaxBin,
                     kWide ? nullptr
                           : reinterpret_cast<const uint32_t *>(((const FinalCtrl *)(wsc + WL.fctrl))->reduced));
        });
        if (e != cudaSuccess) return AHS_ECUDA;
        bases = bucket;
    }

    for (int p = 0; p < passes; p++) {
        PassArgsT<K, V> pa;
        pa.keys_in = src_k;
        pa.vals_in = kv ? src_v : nullptr;
        pa.keys_out = kout;
        pa.vals_out = kv ? d_vals_out : nullptr;
        pa.keys_tmp = tkeys;
        pa.vals_tmp = kv ? tvals : nullptr;
        pa.n = n32;
        pa.pass = (uint32_t)p;
        pa.npasses = (uint32_t)passes;
        pa.shift = count_kv ? 0u : 8u * (uint32_t)p;
        pa.flip = flip;
        pa.sub = umin;
        pa.bucket_base = count_kv ? bases : bases + 256 * p;
        // regions [0, spw) and [spw, 2 spw) of this sort's tile count: both inside the memset
        pa.status = status + (size_t)(p & 1) * status_words_per_pass;
        pa.ticket = tickets + p;
        pa.plan = count_kv ? nullptr : plan;  // K5's plan (no skipping when not enabled)
        pa.status_clear = p + 1 < passes ? status + (size_t)((p + 1) & 1) * status_words_per_pass : nullptr;
        pa.clear_words = p + 1 < passes ? (uint32_t)status_words_per_pass : 0u;
        pa.fault = tickets + kTicketFault;
        void *args[] = {&pa};
        const cudaError_t e = launch(kv ? (count_kv ? KID_COUNT_SCATTER_KV : KID_ONESWEEP_KV) : KID_ONESWEEP, s, [&] {
            cudaLaunchConfig_t cfg;
            cudaLaunchAttribute attr[1];
            pdl_config(cfg, attr, dim3(grid_k6), dim3(k6_block), k6_smem, s);
            cudaLaunchKernelExC(&cfg, k6, args);
        });
        if (e != cudaSuccess) return AHS_ECUDA;
    }
    if (bl_cap) {
        // K10: the bucket-local pass (K9's in-shared-memory stable radix sort, one CTA per bucket, in
        // place on the output; digits all keys of a bucket share are skipped); returns at once when K5
        // chose the classic plan.  It sorts v = key - min, as the digit passes do: a bucket is one
        // feature bin, v >> shift = b, so exactly the low `shift` bits of v differ (ceil(shift / 8)
        // sub-passes); on the key image itself a bin straddles a 2^16 boundary whenever min's low bits
        // are not zero (cfg5 r = 32: ~63 % of the buckets took a third sub-pass)
        cudaError_t le = cudaSuccess;
        const cudaError_t e = launch(KID_BUCKET_SORT, s, [&] {
            const bool ord = di->rank_mode == kRankOrdered;
            if (kv)
                le = seg_launch<K, true>(kout, (const uint32_t *)d_vals_out, kout, (uint32_t *)d_vals_out, n,
                                         bl_offsets, feat->nbins, bl_cap, flip, tickets + kTicketSegBad, ord, s,
                                         plan + kPlanBL, bl_group, umin);
            else
                le = seg_launch<K, false>(kout, nullptr, kout, nullptr, n, bl_offsets, feat->nbins, bl_cap, flip,
                                          tickets + kTicketSegBad, ord, s, plan + kPlanBL, bl_group, umin);
        });
        if (e != cudaSuccess || le != cudaSuccess) return AHS_ECUDA;
    }
    return AHS_OK;
}
}  // namespace

extern "C" {
int ahs_sort(const void *d_keys_in, const uint32_t *d_vals_in, void *d_keys_out, uint32_t *d_vals_out,
             uint64_t n, int32_t strategy, const ahs_features_t *feat, void *d_ws, size_t ws_bytes,
             void *d_tmp, size_t tmp_bytes, void *stream)
{
    return ahs_sort_ex(d_keys_in, d_vals_in, d_keys_out, d_vals_out, n, 4, strategy, feat, d_ws, ws_bytes, d_tmp,
                       tmp_bytes, stream);
}

int ahs_sort_ex(const void *d_keys_in, const void *d_vals_in, void *d_keys_out, void *d_vals_out, uint64_t n,
                uint32_t value_bytes, int32_t strategy, const ahs_features_t *feat, void *d_ws, size_t ws_bytes,
                void *d_tmp, size_t tmp_bytes, void *stream)
{
    if (!feat) return AHS_EINVAL;
    if (strategy != AHS_COUNTING && strategy != AHS_RADIX && strategy != AHS_GENERAL) return AHS_EINVAL;
    const bool kv = d_vals_in != nullptr;
    if (kv && value_bytes != 4 && value_bytes != 8) return AHS_EINVAL;
    if (feat->n != n) return AHS_EFEAT;
    if (n == 0) return AHS_OK;
    if (n > AHS_MAX_N) return AHS_ERANGE;
    const int32_t dtype = (int32_t)feat->dtype;
    if (!dtype_valid(dtype)) return AHS_EFEAT;
    const uintptr_t kal = key_bytes_of(dtype) - 1, val = (kv ? value_bytes : 4) - 1;
    if (!d_keys_in || !d_keys_out || (kv && !d_vals_out) || ((uintptr_t)d_keys_in & kal) ||
        ((uintptr_t)d_keys_out & kal) || (kv && (((uintptr_t)d_vals_in & val) || ((uintptr_t)d_vals_out & val))))
        return AHS_EINVAL;
    if (feat->k == 0 || feat->nbins == 0 || (!dtype_wide(dtype) && feat->k > (1ull << 32))) return AHS_EFEAT;
    cudaStream_t s = (cudaStream_t)stream;
    const bool v64 = kv && value_bytes == 8;
#define AHS_SORT_CALL(K, V)                                                                                   \
    sort_impl<K, V>((const K *)d_keys_in, (const V *)d_vals_in, (K *)d_keys_out, (V *)d_vals_out, n, strategy, \
                    feat, d_ws, ws_bytes, d_tmp, tmp_bytes, s)
    if (dtype_wide(dtype)) return v64 ? AHS_SORT_CALL(uint64_t, uint64_t) : AHS_SORT_CALL(uint64_t, uint32_t);
    return v64 ? AHS_SORT_CALL(uint32_t, uint64_t) : AHS_SORT_CALL(uint32_t, uint32_t);
#undef AHS_SORT_CALL
}

// ------------------------------------------------------------ NEXT-2
int ahs_entropy_sorted(const void *d_keys, uint64_t n, void *d_ws, size_t ws_bytes, double *H, void *stream)
{
    return ahs_entropy_sorted_dtype(d_keys, n, AHS_U32, d_ws, ws_bytes, H, stream);
}

int ahs_entropy_sorted_dtype(const void *d_keys, uint64_t n, int32_t dtype, void *d_ws, size_t ws_bytes, double *H,
                             void *stream)
{
    if (!H) return AHS_EINVAL;
    *H = 0.0;
    if (!dtype_valid(dtype)) return AHS_EINVAL;
    if (n == 0) return AHS_OK;
    if (n > AHS_MAX_N) return AHS_ERANGE;
    if (!d_keys || !d_ws || ((uintptr_t)d_keys & (key_bytes_of(dtype) - 1)) || ((uintptr_t)d_ws & 15u))
        return AHS_EINVAL;
    const bool wide = dtype_wide(dtype);
    const WsLayout L = ws_layout();
    if (ws_bytes < L.total) return AHS_ENOSPACE;
    int sms = 0;
    DevInfo *di = nullptr;
    int rc = device_info(&sms, nullptr, &di);
    if (rc) return rc;
    constexpr uint64_t kTileKeys = (uint64_t)kEntBlock * kEntItems;
    uint64_t grid = std::min<uint64_t>((n + kTileKeys - 1) / kTileKeys, (uint64_t)di->ent_grid[wide ? 1 : 0]);
    grid = std::max<uint64_t>(1, grid);
    uint64_t chunk = (n + grid - 1) / grid;
    constexpr uint64_t kAlign = (uint64_t)kEntItems * (kEntBlock / 32);  // each warp's sub-chunk: 16-key aligned
    chunk = (chunk + kAlign - 1) / kAlign * kAlign;
    grid = (n + chunk - 1) / chunk;
    char *ws = (char *)d_ws;
    RunPieces *pieces = (RunPieces *)(ws + L.ent);
    double *csum = (double *)(ws + L.ent + kEntMaxGrid * sizeof(RunPieces));
    double *dH = csum + kEntMaxGrid;
    uint32_t *done = (uint32_t *)(dH + 1);  // the CTA ticket
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(done, 0, 4, s) != cudaSuccess) return AHS_ECUDA;
    cudaError_t e = launch(KID_ENTROPY_SORTED, s, [&] {
        if (wide)
            launch_k(k_entropy_sorted<kEntBlock, uint64_t>, dim3((unsigned)grid), dim3(kEntBlock), 0, s,
                     (const uint64_t *)d_keys, n, chunk, pieces, csum, dH, done);
        else
            launch_k(k_entropy_sorted<kEntBlock, uint32_t>, dim3((unsigned)grid), dim3(kEntBlock), 0, s,
                     (const uint32_t *)d_keys, n, chunk, pieces, csum, dH, done);
    });
    if (e != cudaSuccess) return AHS_ECUDA;
    if (cudaMemcpyAsync(H, dH, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        cudaGetLastError();
        return AHS_ECUDA;
    }
    return AHS_OK;
}

// -------------------------------------------------------------- host e2e
size_t ahs_host_scratch_bytes_dtype(uint64_t n, int has_vals, int32_t dtype)
{
    if (!dtype_valid(dtype)) return 0;
    const size_t kbytes = key_bytes_of(dtype);
    const size_t kb = align_up(n * kbytes, 256), vb = align_up(n * 4, 256);
    return 2 * kb + (has_vals ? 2 * vb : 0) + ws_layout().total + tmp_layout(n, has_vals, kbytes).total;
}

size_t ahs_host_scratch_bytes(uint64_t n, int has_vals) { return ahs_host_scratch_bytes_dtype(n, has_vals, AHS_U32); }

int ahs_sort_host(const void *h_keys_in, const uint32_t *h_vals_in, void *h_keys_out, uint32_t *h_vals_out,
                  uint64_t n, int32_t dtype, const ahs_thresholds_t *th, void *d_scratch, size_t scratch_bytes,
                  ahs_features_t *feat, int32_t *strategy, int32_t *rule, void *stream)
{
    const int rc = ahs_sort_host_async(h_keys_in, h_vals_in, h_keys_out, h_vals_out, n, dtype, th, d_scratch,
                                       scratch_bytes, feat, strategy, rule, stream);
    if (rc) return rc;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return AHS_ECUDA;
    if (n == 0) return AHS_OK;
    // a look-back that gave up (kTicketFault in the sort's tmp block, same layout as the async call)
    const bool kv = h_vals_in != nullptr;
    const size_t kb = align_up(n * key_bytes_of(dtype), 256), vb = align_up(n * 4, 256);
    const char *tmp = (const char *)d_scratch + 2 * kb + (kv ? 2 * vb : 0) + ws_layout().total;
    uint32_t fault = 0;
    if (cudaMemcpy(&fault, tmp + tmp_layout(0, 0).ticket + kTicketFault * 4, 4, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return AHS_ECUDA;
    return fault ? AHS_ECUDA : AHS_OK;
}

int ahs_sort_host_async(const void *h_keys_in, const uint32_t *h_vals_in, void *h_keys_out, uint32_t *h_vals_out,
                        uint64_t n, int32_t dtype, const ahs_thresholds_t *th, void *d_scratch, size_t scratch_bytes,
                        ahs_features_t *feat, int32_t *strategy, int32_t *rule, void *stream)
{
    if (!dtype_valid(dtype)) return AHS_EINVAL;
    const bool kv = h_vals_in != nullptr;
    if (n > 0 && (!h_keys_in || !h_keys_out || (kv && !h_vals_out) || !d_scratch)) return AHS_EINVAL;
    if (n > AHS_MAX_N) return AHS_ERANGE;
    if (n > 0 && scratch_bytes < ahs_host_scratch_bytes_dtype(n, kv, dtype)) return AHS_ENOSPACE;
    const size_t kbytes = key_bytes_of(dtype);
    if ((uintptr_t)d_scratch & 255u) return AHS_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    ahs_features_t f;
    int32_t st = AHS_COUNTING, ru = AHS_RULE_EMPTY;
    if (n == 0) {
        int rc = ahs_features(nullptr, 0, dtype, nullptr, 0, &f, stream);
        if (rc) return rc;
        rc = ahs_select(&f, th, &st, &ru);
        if (rc) return rc;
    } else {
        const size_t kb = align_up(n * kbytes, 256), vb = align_up(n * 4, 256);
        char *p = (char *)d_scratch;
        void *dk_in = p;
        p += kb;
        void *dk_out = p;
        p += kb;
        uint32_t *dv_in = nullptr, *dv_out = nullptr;
        if (kv) {
            dv_in = (uint32_t *)p;
            p += vb;
            dv_out = (uint32_t *)p;
            p += vb;
        }
        void *ws = p;
        p += ws_layout().total;
        void *tmp = p;
        const size_t tmpb = tmp_layout(n, kv, kbytes).total;
        if (cudaMemcpyAsync(dk_in, h_keys_in, n * kbytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return AHS_ECUDA;
        if (kv && cudaMemcpyAsync(dv_in, h_vals_in, n * 4, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return AHS_ECUDA;
        int rc = ahs_features(dk_in, n, dtype, ws, ws_layout().total, &f, stream);
        if (rc) return rc;
        rc = ahs_select(&f, th, &st, &ru);
        if (rc) return rc;
        rc = ahs_sort(dk_in, dv_in, dk_out, dv_out, n, st, &f, ws, ws_layout().total, tmp, tmpb, stream);
        if (rc) return rc;
        if (cudaMemcpyAsync(h_keys_out, dk_out, n * kbytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return AHS_ECUDA;
        if (kv && cudaMemcpyAsync(h_vals_out, dv_out, n * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return AHS_ECUDA;
    }
    if (feat) *feat = f;
    if (strategy) *strategy = st;
    if (rule) *rule = ru;
    return AHS_OK;
}

// --------------------------------------------------- segment sort (NEXT-4)
}  // extern "C"
namespace {
// Opt-in dynamic shared memory above 48 KiB is a per-device function attribute: set it once per
// (kernel, device) pair.  A failure is returned (and not cached), so the caller reports it.
cudaError_t opt_in_smem(const void *fn, size_t smem)
{
    if (smem <= 48u * 1024u) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    done.insert({fn, dev});
    return cudaSuccess;
}

template <typename K, bool KV, int L>
cudaError_t seg_small(const void *kin, const uint32_t *vin, void *kout, uint32_t *vout, uint64_t n,
                      const uint32_t *offsets, uint32_t nseg, uint32_t max_segment, K flip, uint32_t *bad,
                      cudaStream_t s)
{
    constexpr size_t smem = seg_small_smem<K, KV>();
    const cudaError_t ae = opt_in_smem((const void *)k_seg_small<K, KV, L>, smem);
    if (ae != cudaSuccess) return ae;
    const unsigned g = (nseg + kSegSmallBlock - 1) / kSegSmallBlock;
    return launch_k(k_seg_small<K, KV, L>, dim3(g), dim3(kSegSmallBlock), smem, s, (const K *)kin, vin, (K *)kout,
                    vout, offsets, nseg, n, flip, max_segment, bad);
}

// K10 (bucket.cuh): one CTA of BLOCK threads per segment of <= BLOCK IPT keys, ordered ranking
template <typename K, bool KV, int IPT, int BLOCK = 256>
cudaError_t seg_bucket(const void *kin, const uint32_t *vin, void *kout, uint32_t *vout, uint64_t n,
                       const uint32_t *offsets, uint32_t nseg, K flip, K sub, uint32_t *bad, cudaStream_t s,
                       const uint32_t *gate, uint32_t group)
{
    using BS = BucketSort<K, KV, IPT, BLOCK>;
#ifndef AHS_K10_MINB16
#define AHS_K10_MINB16 4  // 64 registers (12-32 B of spill), 4 CTAs per SM: cfg5_r32 bucket pass 1923 -> 1863 us
#endif
    // 256 threads: 64 registers at 4 CTAs per SM up to 18 keys per thread; 128 threads: 8 CTAs
    constexpr int MINB = BLOCK == 128 ? 8 : (IPT >= 32 ? 2 : (IPT >= 20 ? 3 : (IPT >= 16 ? AHS_K10_MINB16 : 4)));
    const cudaError_t ae = opt_in_smem((const void *)k_bucket_sort<K, KV, IPT, MINB, BLOCK>, BS::kSmem);
    if (ae != cudaSuccess) return ae;
    const unsigned grid = (unsigned)((nseg + group - 1) / group);
    return launch_k(k_bucket_sort<K, KV, IPT, MINB, BLOCK>, dim3(grid), dim3(BLOCK), BS::kSmem, s, (const K *)kin,
                    vin, (K *)kout, vout, offsets, nseg, n, flip, sub, bad, gate, group);
}

template <typename K, bool KV, int GROUP, int CAP, bool ORD>
cudaError_t seg_radix(const void *kin, const uint32_t *vin, void *kout, uint32_t *vout, uint64_t n,
                      const uint32_t *offsets, uint32_t nseg, uint32_t max_segment, K flip, uint32_t *bad,
                      cudaStream_t s, const uint32_t *gate = nullptr, K sub = 0)
{
    constexpr size_t smem = seg_radix_smem<K, KV, GROUP, CAP>();
    const cudaError_t ae = opt_in_smem((const void *)k_seg_radix<K, KV, GROUP, CAP, ORD>, smem);
    if (ae != cudaSuccess) return ae;
    return launch_k(k_seg_radix<K, KV, GROUP, CAP, ORD>, dim3(nseg), dim3(GROUP), smem,
                    s, (const K *)kin, vin, (K *)kout, vout, offsets, nseg, n, flip, sub, max_segment, bad, gate);
}

// register network length / CTA size from the declared maximum segment
template <typename K, bool KV>
cudaError_t seg_launch(const void *kin, const uint32_t *vin, void *kout, uint32_t *vout, uint64_t n,
                       const uint32_t *offsets, uint32_t nseg, uint32_t max_segment, K flip, uint32_t *bad,
                       bool ord, cudaStream_t s, const uint32_t *gate, uint32_t group, K sub)
{
#define AHS_SEG_ARGS kin, vin, kout, vout, n, offsets, nseg, max_segment, flip, bad, s
    if (max_segment <= 8) return seg_small<K, KV, 8>(AHS_SEG_ARGS);
    if (max_segment <= 16) return seg_small<K, KV, 16>(AHS_SEG_ARGS);
    if (max_segment <= 20) return seg_small<K, KV, 20>(AHS_SEG_ARGS);  // the paper's n <= 20 Insertion branch
    if (max_segment <= 24) return seg_small<K, KV, 24>(AHS_SEG_ARGS);
    if (max_segment <= (uint32_t)kSegSmallMax) return seg_small<K, KV, 32>(AHS_SEG_ARGS);
    // K9r: threads per segment from the declared maximum (16 keys per thread, one
    // warp up to 512 keys); the ordered ranking when the device passed its self-test
    if (ord && (group > 1 || (g_k10.load(std::memory_order_relaxed) && max_segment > 512))) {
        // K10: 128 or 256 threads per segment, keys in registers between the passes (faster than K9r
        // above 512 keys; slower below, profiles/r02_summary.md)
#define AHS_BK_ARGS kin, vin, kout, vout, n, offsets, nseg, flip, sub, bad, s, gate, group
        // 128 x 8 from 513 keys (2^14 segments of 600-1024 keys: 137.2 -> 118.8 us against K9r, pairs
        // 192.5 -> 145.4, uint64 325.6 -> 268.3); K9r below (300-512 keys: K10 131.1 -> 153.6 us)
        if (max_segment <= 1024) return seg_bucket<K, KV, 8, 128>(AHS_BK_ARGS);
        if (max_segment <= 1536) return seg_bucket<K, KV, 12, 128>(AHS_BK_ARGS);
        // 128 threads up to 2048 keys (2^13 segments of 1000-2048 keys: 122.6 -> 102.1 us against
        // 256 x 8, pairs 147.5 -> 135.1, uint64 270.2 -> 249.5; profiles/r02_summary.md)
        if (max_segment <= 2048) return seg_bucket<K, KV, 16, 128>(AHS_BK_ARGS);
        if (max_segment <= 4096) return seg_bucket<K, KV, 16>(AHS_BK_ARGS);
        if (max_segment <= 4608) return seg_bucket<K, KV, 18>(AHS_BK_ARGS);
        if (max_segment <= 5120) return seg_bucket<K, KV, 20>(AHS_BK_ARGS);
        if (max_segment <= 6144) return seg_bucket<K, KV, 24>(AHS_BK_ARGS);
        return seg_bucket<K, KV, 32>(AHS_BK_ARGS);
#undef AHS_BK_ARGS
    }
    if (ord) {
        if (max_segment <= 256) return seg_radix<K, KV, 32, 256, true>(AHS_SEG_ARGS, gate, sub);
        if (max_segment <= 512) return seg_radix<K, KV, 32, 512, true>(AHS_SEG_ARGS, gate, sub);
        if (max_segment <= 1024) return seg_radix<K, KV, 64, 1024, true>(AHS_SEG_ARGS, gate, sub);
        if (max_segment <= 2048) return seg_radix<K, KV, 128, 2048, true>(AHS_SEG_ARGS, gate, sub);
        if (max_segment <= 4096) return seg_radix<K, KV, 256, 4096, true>(AHS_SEG_ARGS, gate, sub);
        return seg_radix<K, KV, 512, 8192, true>(AHS_SEG_ARGS, gate, sub);
    }
    if (max_segment <= 256) return seg_radix<K, KV, 32, 256, false>(AHS_SEG_ARGS, gate, sub);
    if (max_segment <= 512) return seg_radix<K, KV, 32, 512, false>(AHS_SEG_ARGS, gate, sub);
    if (max_segment <= 1024) return seg_radix<K, KV, 64, 1024, false>(AHS_SEG_ARGS, gate, sub);
    if (max_segment <= 2048) return seg_radix<K, KV, 128, 2048, false>(AHS_SEG_ARGS, gate, sub);
    if (max_segment <= 4096) return seg_radix<K, KV, 256, 4096, false>(AHS_SEG_ARGS, gate, sub);
    return seg_radix<K, KV, 512, 8192, false>(AHS_SEG_ARGS, gate, sub);
#undef AHS_SEG_ARGS
}
}  // namespace
extern "C" {

int ahs_sort_segments(const void *d_keys_in, const uint32_t *d_vals_in, void *d_keys_out, uint32_t *d_vals_out,
                      uint64_t n, const uint32_t *d_offsets, uint32_t num_segments, uint32_t max_segment,
                      int32_t dtype, uint32_t *d_bad, void *stream)
{
    if (!dtype_valid(dtype)) return AHS_EINVAL;
    if (max_segment > (uint32_t)kSegMedMax) return AHS_ERANGE;
    if (n > AHS_MAX_N) return AHS_ERANGE;
    const bool kv = d_vals_in != nullptr;
    const uintptr_t kal = key_bytes_of(dtype) - 1;
    if (!d_bad || (num_segments > 0 && (!d_offsets || !d_keys_in || !d_keys_out || (kv && !d_vals_out))) ||
        ((uintptr_t)d_keys_in & kal) || ((uintptr_t)d_keys_out & kal))
        return AHS_EINVAL;
    int sms = 0;
    DevInfo *di = nullptr;
    int rc = device_info(&sms, nullptr, &di);
    if (rc) return rc;
    const bool ord = di->rank_mode == kRankOrdered;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(d_bad, 0, 4, s) != cudaSuccess) return AHS_ECUDA;
    if (num_segments == 0) return AHS_OK;
    cudaError_t le = cudaSuccess;  // seg_launch's own status (attribute set-up, launch)
    const cudaError_t e = launch(KID_SEG_SORT, s, [&] {
        if (dtype_wide(dtype)) {
            const uint64_t flip = flip64_of(dtype);
            if (kv) le = seg_launch<uint64_t, true>(d_keys_in, d_vals_in, d_keys_out, d_vals_out, n, d_offsets,
                                                    num_segments, max_segment, flip, d_bad, ord, s);
            else le = seg_launch<uint64_t, false>(d_keys_in, nullptr, d_keys_out, nullptr, n, d_offsets,
                                                  num_segments, max_segment, flip, d_bad, ord, s);
        } else {
            const uint32_t flip = flip_of(dtype);
            if (kv) le = seg_launch<uint32_t, true>(d_keys_in, d_vals_in, d_keys_out, d_vals_out, n, d_offsets,
                                                    num_segments, max_segment, flip, d_bad, ord, s);
            else le = seg_launch<uint32_t, false>(d_keys_in, nullptr, d_keys_out, nullptr, n, d_offsets,
                                                  num_segments, max_segment, flip, d_bad, ord, s);
        }
    });
    return (e == cudaSuccess && le == cudaSuccess) ? AHS_OK : AHS_ECUDA;
}

// ------------------------------------------------------ classifier (NEXT-4)
}  // extern "C"
struct ahs_model {
    ahs::model::Model m;
};
extern "C" {

int ahs_model_load(const char *json, size_t len, ahs_model_t **model, char *err, size_t err_len)
{
    if (err && err_len) err[0] = 0;
    if (!json || !model) return AHS_EINVAL;
    *model = nullptr;
    std::unique_ptr<ahs_model> h(new (std::nothrow) ahs_model());
    if (!h) return AHS_EINVAL;
    std::string msg;
    const ahs::model::LoadStatus st = ahs::model::load(json, len, h->m, msg);
    if (st != ahs::model::LOAD_OK) {
        if (err && err_len) std::snprintf(err, err_len, "%s", msg.c_str());
        return st == ahs::model::LOAD_VERSION ? AHS_EMODELVER : AHS_EMODEL;
    }
    *model = h.release();
    return AHS_OK;
}

void ahs_model_free(ahs_model_t *model) { delete model; }

int ahs_model_predict(const ahs_model_t *model, double n, double k, double H, int32_t *algo4, double *scores4)
{
    if (!model || !algo4) return AHS_EINVAL;
    double sc[4];
    *algo4 = model->m.predict(n, k, H, sc);
    if (scores4)
        for (int c = 0; c < 4; c++) scores4[c] = sc[c];
    return AHS_OK;
}

int ahs_select_model(const ahs_features_t *feat, const ahs_thresholds_t *th, const ahs_model_t *model,
                     uint64_t ml_min_n, int32_t *strategy, int32_t *rule, int32_t *source)
{
    if (!feat || !strategy) return AHS_EINVAL;
    if (source) *source = 0;
    if (!model || feat->n == 0 || feat->k == 1 || feat->n < ml_min_n)  // P:411 shortcuts, then Table IV's n range
        return ahs_select(feat, th, strategy, rule);
    if (th) {  // the thresholds are still validated (they govern the fallback path)
        int32_t s0, r0;
        const int rc = ahs_select(feat, th, &s0, &r0);
        if (rc) return rc;
    }
    int32_t a = 0;
    ahs_model_predict(model, (double)feat->n, (double)feat->k, feat->entropy, &a, nullptr);
    *strategy = a == ahs::model::COUNTING ? AHS_COUNTING : a == ahs::model::RADIX ? AHS_RADIX : AHS_GENERAL;
    if (rule) *rule = AHS_RULE_MODEL;
    if (source) *source = 1;
    return AHS_OK;
}

}  // extern "C"
