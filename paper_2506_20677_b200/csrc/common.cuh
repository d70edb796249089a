// common.cuh — device-side helpers shared by the libahs kernels (sm_100a only).
//
// Key space: every kernel works on the ORDERED image u = key ^ flip of a key
// (flip = 0x80000000 for int32, 0 for uint32), so unsigned comparison of u is
// the key's own order and u - u_min = key - min (mod 2^32).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ahs {

constexpr uint32_t kFull = 0xffffffffu;

// Per-block result of K1 feat_reduce (ws); reduced again by K2 and K3.
struct Partial {
    uint32_t mn, mx;   // ordered space
    uint64_t desc;
    uint32_t an, orv;  // AND and OR of the ordered images: bits every key shares (K5's digit placement)
};
static_assert(sizeof(Partial) == 24, "Partial: mn, mx, desc, an, orv");

// Device-side feature record, written by K3 into ws and into the host's
// mapped buffer (seq last).  umin/umax: ordered images (32-bit keys zero-extended).
struct DevFeatures {
    uint64_t umin, umax;
    uint64_t descents;
    uint64_t k;                       // saturated at 2^64 - 1 (64-bit keys spanning the range)
    uint32_t bits, shift, nb, nparts; // nparts: K1 CTA count (rows of the low-byte histograms)
    double entropy;
    uint32_t nrows2, ksat;            // nrows2: K2 CTA count (rows of the digit-1 histograms)
    uint64_t seq;                     // the host polls this word
};
static_assert(sizeof(DevFeatures) == 72, "DevFeatures is 72 bytes (9 words, seq last)");

// 64-bit keys (NEXT-3): per-block result of K1 (ordered images)
struct Partial64 {
    uint64_t mn, mx;
    uint64_t desc;
};

// Derived range quantities (§III.A line 96 k = max - min + 1;
// DESIGN.md R1: shift = max(0, bitlen(k-1) - 16), nb = ((k-1) >> shift) + 1).
struct Range {
    uint64_t k;
    uint32_t bits, shift, nb;
};

__host__ __device__ __forceinline__ Range derive_range(uint32_t umin, uint32_t umax, uint32_t entropy_bits)
{
    Range r;
    r.k = (uint64_t)(umax - umin) + 1ull;
    uint64_t km1 = r.k - 1ull;
#ifdef __CUDA_ARCH__
    r.bits = km1 ? 64u - (uint32_t)__clzll((long long)km1) : 0u;
#else
    r.bits = 0;
    while (km1 >> r.bits) r.bits++;
#endif
    r.shift = r.bits > entropy_bits ? r.bits - entropy_bits : 0u;
    r.nb = (uint32_t)(((r.k - 1ull) >> r.shift) + 1ull);
    return r;
}

// ------------------------------------------- programmatic dependent launch
// Every libahs kernel starts with pdl_begin(): wait until the previous grid in
// the stream has completed and its memory is visible (a no-op unless launched
// with programmatic stream serialization), then let the next grid launch: its
// CTAs become resident as resources free up and wait in their own pdl_begin(),
// which hides the launch latency between the kernels of a step.  Nothing
// touches global memory before the wait.
__device__ __forceinline__ void pdl_begin()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// 64-bit keys: k = umax - umin + 1 can be 2^64: reported saturated
struct Range64 {
    uint64_t k;
    uint32_t bits, shift, nb, ksat;
};

__host__ __device__ __forceinline__ Range64 derive_range64(uint64_t umin, uint64_t umax, uint32_t entropy_bits)
{
    Range64 r;
    const uint64_t km1 = umax - umin;
    r.ksat = km1 == ~0ull ? 1u : 0u;
    r.k = r.ksat ? km1 : km1 + 1ull;
#ifdef __CUDA_ARCH__
    r.bits = km1 ? 64u - (uint32_t)__clzll((long long)km1) : 0u;
#else
    r.bits = 0;
    while (r.bits < 64 && (km1 >> r.bits)) r.bits++;
#endif
    r.shift = r.bits > entropy_bits ? r.bits - entropy_bits : 0u;
    r.nb = (uint32_t)((km1 >> r.shift) + 1ull);
    return r;
}

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ uint4 ld_nc_v4(const uint4 *p)
{
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t ld_nc(const uint32_t *p)
{
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ uint64_t ld_nc(const uint64_t *p)
{
    uint64_t r;
    asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p)
{
    uint32_t r;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}

__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v)
{
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_cs_v4(uint4 *p, uint4 v)
{
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ------------------------------------------------ TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// 1-D bulk copy global -> shared (TMA), completion signalled on `bar`.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// order this thread's earlier generic-proxy shared-memory accesses (made
// visible to it by a barrier) before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Streaming reader: the 16-byte-aligned body of the key array (nvec uint4
// vectors) in chunks of CHUNK bytes; CTA b consumes chunks b, b + G, ...
// Thread 0 keeps STAGES chunks in flight with TMA bulk copies (each chunk
// buffer also receives the 16 bytes after the chunk when they exist, so a
// consumer can see the successor of the chunk's last key); all threads wait
// on the chunk's mbarrier, call consume(chunk_smem, nv, v0) and meet at a
// barrier before the buffer is refilled.  Memory-level parallelism is
// STAGES * CHUNK bytes per CTA independent of register pressure.
// REV: the chunks are visited last to first (chunk nchunks - 1 - (b + i * G)), so a
// pass that follows a forward pass over the same keys starts on the chunks that
// pass read last, which are still in L2, and leaves the first chunks in L2 for
// the sort's first digit pass.
template <int STAGES, int CHUNK, bool REV = false, typename F>
__device__ __forceinline__ void stream_chunks(const uint4 *__restrict__ body, uint64_t nvec, uint8_t *buf,
                                              uint64_t *bars, F &&consume)
{
    constexpr uint32_t VPC = CHUNK / 16;
    constexpr uint32_t STRIDE = CHUNK + 16;
    const uint32_t nchunks = (uint32_t)((nvec + VPC - 1) / VPC);
    const uint32_t mine = blockIdx.x < nchunks ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) mbar_init(&bars[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto chunk = [&](uint32_t i) -> uint64_t {
        const uint32_t c = blockIdx.x + i * gridDim.x;
        return REV ? nchunks - 1u - c : c;
    };
    auto issue = [&](uint32_t i, uint32_t s) {
        const uint64_t v0 = chunk(i) * VPC;
        const uint64_t nv = min((uint64_t)VPC, nvec - v0);
        const uint64_t ncopy = min(nv + 1, nvec - v0);  // + successor vector when it exists
        mbar_expect_tx(&bars[s], (uint32_t)(ncopy * 16));
        tma_load_1d(buf + s * STRIDE, body + v0, (uint32_t)(ncopy * 16), &bars[s]);
    };
    if (threadIdx.x == 0)
        for (uint32_t i = 0; i < (uint32_t)STAGES && i < mine; i++) issue(i, i);
    uint32_t s = 0, phase = 0;
    for (uint32_t i = 0; i < mine; i++) {
        mbar_wait(&bars[s], phase);
        const uint64_t v0 = chunk(i) * VPC;
        const uint32_t nv = (uint32_t)min((uint64_t)VPC, nvec - v0);
        consume(reinterpret_cast<const uint4 *>(buf + s * STRIDE), nv, v0);
        __syncthreads();
        if (threadIdx.x == 0 && i + STAGES < mine) {
            fence_proxy_async();
            issue(i + STAGES, s);
        }
        if (++s == (uint32_t)STAGES) {
            s = 0;
            phase ^= 1u;
        }
    }
}

// Split of a 4-byte-aligned key array into an unaligned head (< 4 keys), a
// 16-byte-aligned body of uint4 vectors, and a tail (< 4 keys).
struct VecSplit {
    uint64_t head, nvec, tail0;
};

__device__ __forceinline__ VecSplit vec_split(const uint32_t *p, uint64_t n)
{
    VecSplit s;
    uint64_t mis = ((16u - ((uintptr_t)p & 15u)) & 15u) >> 2;
    s.head = mis < n ? mis : n;
    s.nvec = (n - s.head) >> 2;
    s.tail0 = s.head + 4ull * s.nvec;
    return s;
}

// Visit every key once with warp-uniform calls op(u, active) where
// u = key ^ flip.  All 32 lanes of a warp call op together (so op may use
// warp collectives); inactive lanes pass active = false.  Body: uint4
// streaming loads, UNROLL vectors in flight per thread, grid-stride.
// Head/tail (<= 6 keys): warp 0 of block 0.
template <int UNROLL, typename Op>
__device__ __forceinline__ void for_each_key(const uint32_t *__restrict__ keys, uint64_t n,
                                             uint32_t flip, Op &op)
{
    const VecSplit sp = vec_split(keys, n);
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint4 *vp = reinterpret_cast<const uint4 *>(keys + sp.head);
    for (uint64_t vb = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); vb < sp.nvec;
         vb += stride * UNROLL) {
        uint4 x[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            uint64_t v = vb + (uint64_t)u * stride + lane;
            x[u] = v < sp.nvec ? ld_nc_v4(vp + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            uint64_t v = vb + (uint64_t)u * stride + lane;
            bool act = v < sp.nvec;
            op(x[u].x ^ flip, act);
            op(x[u].y ^ flip, act);
            op(x[u].z ^ flip, act);
            op(x[u].w ^ flip, act);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        uint64_t i = lane < 3 ? lane : sp.tail0 + (lane - 3);
        bool act = lane < 3 ? i < sp.head : (lane < 6 && i < n);
        uint32_t u = act ? (keys[i] ^ flip) : 0u;
        op(u, act);
    }
}

}  // namespace ahs
