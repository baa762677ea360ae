// common.cuh — device helpers shared by the libbs.so kernels (sm_100a).
// Nothing here is shared with oracle/ (the oracle is an independent C file).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bs {

// host: counts this library's kernel launches on the lookup paths (bs_launch_count)
void count_launch();

template <class K> struct KeyMax;
template <> struct KeyMax<uint32_t> { static constexpr uint32_t v = 0xFFFFFFFFu; };
template <> struct KeyMax<uint64_t> { static constexpr uint64_t v = 0xFFFFFFFFFFFFFFFFull; };

// LPOW2(n): largest power of two <= n, via count-leading-zeros.  n >= 1.
__host__ __device__ __forceinline__ uint64_t lpow2(uint64_t n) {
#ifdef __CUDA_ARCH__
    return 1ull << (63 - __clzll((long long)n));
#else
    return 1ull << (63 - __builtin_clzll(n));
#endif
}

// Result word (include/bs.h RESULT CONTRACT).  `v` is the value of the entry
// at `off` (the last taken probe, or a[n-1] if no step was taken); after the
// offset search `off` is the first entry >= q or n-1, so lb = off if
// v >= q else n, and the lookup hits iff v == q.
template <class O, class K>
__device__ __forceinline__ O encode(uint64_t off, K v, K q, uint64_t n) {
    const uint64_t lb = (v >= q) ? off : n;
    constexpr uint64_t MISS = 1ull << (8 * sizeof(O) - 1);
    return (O)((v == q) ? lb : (lb | MISS));
}

// ---------------------------------------------------------------- cache policies
// L2 eviction-priority policies (createpolicy, sm_80+), used with
// ld/st .L2::cache_hint.  evict_first for streamed queries/results and for
// the deepest probes so they do not evict the upper search levels.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// read-only global loads: plain / with L2 cache hint (+ no L1 allocation for streams)
__device__ __forceinline__ uint64_t ldg(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t ldg_hint(const uint64_t* p, uint64_t pol) {
    uint64_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldg_hint(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint64_t ldg_stream(const uint64_t* p, uint64_t pol) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void stg_stream(uint64_t* p, uint64_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_stream(uint32_t* p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;" :: "l"(p), "r"(v), "l"(pol) : "memory");
}

// Random-access loads that do NOT allocate in L1: a plain ld.global.nc miss
// makes L1 request the whole 128-B line from L2 (measured: 3.6 L2 sectors and
// ~110 DRAM bytes per random 8-B load, tools/ubench_gather.cu), while
// .L1::no_allocate requests only the touched sectors.
__device__ __forceinline__ uint64_t ld_na(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_na(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t ld_na_hint(const uint64_t* p, uint64_t pol) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_na_hint(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// Random probe of the sorted array / separator levels (no L1 allocation),
// optionally with an L2 eviction-priority policy (uniform branch).
template <class K>
__device__ __forceinline__ K load_key(const K* p, bool hinted, uint64_t pol) {
    return hinted ? ld_na_hint(p, pol) : ld_na(p);
}
template <class K>
__device__ __forceinline__ K load_stream(const K* p, bool hinted, uint64_t pol) {
    return hinted ? ldg_stream(p, pol) : ldg(p);
}
template <class O>
__device__ __forceinline__ void store_stream(O* p, O v, bool hinted, uint64_t pol) {
    if (hinted) stg_stream(p, v, pol);
    else *p = v;
}

// ---------------------------------------------------------------- TMA bulk copy
// cp.async.bulk global -> shared completed on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// 4-B shared load from a shared-window address (volatile: stays after the
// staging barrier; the table is read-only once staged)
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}

// Stage `bytes` (multiple of 16, both addresses 16-B aligned) from global into
// shared memory with TMA bulk copies issued by one thread; every thread of the
// CTA returns once the bytes have landed.  `bar` is a CTA-shared mbarrier.
__device__ __forceinline__ void stage_to_smem(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    if (bytes % 16u != 0u) __trap();   // bulk copies move 16-B multiples; never wait forever
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, bytes);
        constexpr uint32_t CH = 32768;
        for (uint32_t o = 0; o < bytes; o += CH) {
            const uint32_t b = (bytes - o < CH) ? (bytes - o) : CH;
            bulk_g2s((char*)dst + o, (const char*)src + o, b, bar);
        }
    }
    mbar_wait(bar, 0);
}

}  // namespace bs
