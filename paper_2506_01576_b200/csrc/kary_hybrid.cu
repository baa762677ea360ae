// kary_hybrid.cu — K-ary search (§5), B200 hybrid schedule.
//
// Same index as kary.cu (chunk-max separators, top-first levels of W-slot
// nodes, child m*K+j, leaf = the unpermuted sorted array; reading R16) and the
// same result, but the work of one lookup is split by where its data lives:
//
//  * shared-memory levels (the top Ls levels, staged once per CTA by TMA, the
//    §5.1 "pinning" of KS): ONE thread per lookup.  The thread reads its
//    node's W slots with 16-B shared loads and counts separators < q.  No
//    cross-lane traffic, 32 lookups per warp instruction.
//  * global levels + leaf (L2 / HBM): W lanes per lookup ("K-1 threads
//    compare in parallel"), so each node / leaf is ONE coalesced line request
//    (an L2 miss costs a 128-B line whatever is read).  A warp's 32 lookups
//    are handed to its 32/W groups in W waves (__shfl_sync), I waves in
//    flight at a time; __ballot_sync + __popc pick the child; the leaf is read
//    with vector loads (CPL = C/W keys per lane) and reduced with __shfl_xor.
//  * results are shuffled back to the owning lane and stored coalesced; the
//    next warp-tile's queries are prefetched during the descent.
#include "common.cuh"
#include "params.h"

namespace bs {

__device__ __forceinline__ void ld_na_v2(const uint64_t* p, bool hint, uint64_t pol, uint64_t& a, uint64_t& b) {
    if (hint)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                     : "=l"(a), "=l"(b) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ void ld_na_v2(const uint32_t* p, bool hint, uint64_t pol, uint32_t& a, uint32_t& b) {
    if (hint)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                     : "=r"(a), "=r"(b) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p));
}

// count of the W slots of a shared-memory node that are < key
template <class K, int W>
__device__ __forceinline__ uint32_t smem_node_count(const K* nd, K key) {
    uint32_t c = 0;
    if constexpr ((W * sizeof(K)) % 16 == 0) {
        const uint4* v = reinterpret_cast<const uint4*>(nd);
#pragma unroll
        for (int t = 0; t < (int)(W * sizeof(K) / 16); ++t) {
            const uint4 x = v[t];
            if constexpr (sizeof(K) == 8) {
                const uint64_t a = ((uint64_t)x.y << 32) | x.x, b = ((uint64_t)x.w << 32) | x.z;
                c += (a < (uint64_t)key) + (b < (uint64_t)key);
            } else {
                c += (x.x < (uint32_t)key) + (x.y < (uint32_t)key) + (x.z < (uint32_t)key) + (x.w < (uint32_t)key);
            }
        }
    } else {
#pragma unroll
        for (int t = 0; t < W; ++t) c += nd[t] < key;
    }
    return c;
}

template <class K, class O, int W, int I, int CPL>
__global__ void k_kary_hybrid(const KaryParams<K> p, const K* __restrict__ q, uint64_t m, O* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    K* S = reinterpret_cast<K*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.smem_bytes);
    constexpr int GPW = 32 / W;
    constexpr uint32_t GMASK = (W == 32) ? 0xFFFFFFFFu : ((1u << W) - 1u);
    static_assert(W % I == 0, "I must divide W");
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t j = lane & (W - 1);
    const uint32_t g = lane / W;
    const uint32_t gshift = g * W;
    const uint32_t my_r = lane / GPW, my_gl = (lane % GPW) * W;   // my lookup's wave and its group's first lane

    if (p.smem_bytes) stage_to_smem(S, p.sep, p.smem_bytes, bar);

    const uint64_t pol_first = policy_evict_first();
    const uint64_t pol_last = policy_evict_last();
    const bool sh = p.stream_hint != 0, lh = p.leaf_hint != 0, sep_last = p.sep_hint != 0;
    const uint64_t n = p.n;
    const uint32_t K_ = p.K, C = p.C, L = p.L, Ls = p.Ls;
    const uint64_t warps_total = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nwt = (m + 31) / 32;
    uint64_t wt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    K knext = KeyMax<K>::v;
    if (wt < nwt && wt * 32 + lane < m) knext = load_stream(q + wt * 32 + lane, sh, pol_first);

    for (; wt < nwt; wt += warps_total) {
        const K key = knext;
        {
            const uint64_t wn = wt + warps_total;
            const uint64_t i = wn * 32 + lane;
            knext = (wn < nwt && i < m) ? load_stream(q + i, sh, pol_first) : KeyMax<K>::v;
        }
        // ---- shared-memory levels: one thread per lookup ----
        uint32_t node = 0;
        for (uint32_t l = 0; l < Ls; ++l) {
            const uint32_t cnt = smem_node_count<K, W>(S + p.lvl_base[l] + (uint64_t)node * W, key);
            const uint32_t child = node * K_ + cnt;
            const uint32_t last = p.nodes_next[l] - 1;
            node = child < last ? child : last;
        }
        // ---- global levels + leaf: W lanes per lookup, I waves in flight ----
        O mine = 0;
#pragma unroll 1
        for (int b = 0; b < W / I; ++b) {
            K kk[I];
            uint32_t nn[I];
#pragma unroll
            for (int i = 0; i < I; ++i) {
                const int src = (b * I + i) * GPW + (int)g;
                kk[i] = __shfl_sync(0xFFFFFFFFu, key, src);
                nn[i] = __shfl_sync(0xFFFFFFFFu, node, src);
            }
            for (uint32_t l = Ls; l < L; ++l) {
                const K* lv = p.sep + p.lvl_base[l];
                K s[I];
                if (sep_last) {
#pragma unroll
                    for (int i = 0; i < I; ++i) s[i] = ld_na_hint(lv + (uint64_t)nn[i] * W + j, pol_last);
                } else {
#pragma unroll
                    for (int i = 0; i < I; ++i) s[i] = ld_na(lv + (uint64_t)nn[i] * W + j);
                }
                const uint32_t last = p.nodes_next[l] - 1;
#pragma unroll
                for (int i = 0; i < I; ++i) {
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, s[i] < kk[i]);
                    const uint32_t child = nn[i] * K_ + __popc((bal >> gshift) & GMASK);
                    nn[i] = child < last ? child : last;
                }
            }
            // leaf chunk: lane j holds keys [c*C + j*CPL, +CPL)  (array padded past n with MAX)
            K x[I][CPL];
#pragma unroll
            for (int i = 0; i < I; ++i) {
                const K* lp = p.a + (uint64_t)nn[i] * C + j * CPL;
                if (j * CPL < C) {
                    if constexpr (CPL == 1) {
                        x[i][0] = load_key(lp, lh, pol_first);
                    } else {
#pragma unroll
                        for (int t = 0; t < CPL; t += 2) ld_na_v2(lp + t, lh, pol_first, x[i][t], x[i][t + 1]);
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < CPL; ++t) x[i][t] = KeyMax<K>::v;
                }
            }
#pragma unroll
            for (int i = 0; i < I; ++i) {
                const uint64_t p0 = (uint64_t)nn[i] * C + j * CPL;
                uint32_t lt = 0, eq = 0;
#pragma unroll
                for (int t = 0; t < CPL; ++t) {
                    const bool ok = (j * CPL + t < C) && (p0 + t < n);
                    lt += (ok && x[i][t] < kk[i]) ? 1u : 0u;
                    eq |= (ok && x[i][t] == kk[i]) ? 1u : 0u;
                }
#pragma unroll
                for (int o = W / 2; o > 0; o >>= 1) lt += __shfl_xor_sync(0xFFFFFFFFu, lt, o);
                const uint32_t hit = (__ballot_sync(0xFFFFFFFFu, eq != 0) >> gshift) & GMASK;
                uint64_t lbv = (uint64_t)nn[i] * C + lt;
                if (lbv > n) lbv = n;
                constexpr uint64_t MISS = 1ull << (8 * sizeof(O) - 1);
                const O res = (O)(hit ? lbv : (lbv | MISS));
                const O v = __shfl_sync(0xFFFFFFFFu, res, my_gl);
                if ((int)my_r == b * I + i) mine = v;
            }
        }
        const uint64_t i = wt * 32 + lane;
        if (i < m) store_stream(out + i, mine, sh, pol_first);
    }
}

template <class K, class O, int W, int I, int CPL>
static cudaError_t go_hybrid(const void* params, const void* q, uint64_t m, void* out, uint32_t threads,
                             Grid grid, uint32_t smem, cudaStream_t s, bool* uns) {
    auto kern = k_kary_hybrid<K, O, W, I, CPL>;
    const uint64_t per_cta = (uint64_t)threads;   // one lookup per thread per tile
    const uint64_t need = (m + per_cta - 1) / per_cta;
    uint64_t g = 0;
    cudaError_t e = plan_grid((const void*)kern, threads, smem, grid, need, carveout_for(smem, threads), &g, uns);
    if (e != cudaSuccess || *uns) return e;
    kern<<<(unsigned)g, threads, smem, s>>>(*(const KaryParams<K>*)params, (const K*)q, m, (O*)out);
    count_launch();
    return cudaGetLastError();
}

template <class K, class O, int W>
static cudaError_t hybrid_w(const void* params, const void* q, uint64_t m, void* out, uint32_t threads,
                            uint32_t I, uint32_t cpl, Grid grid, uint32_t smem, cudaStream_t s, bool* uns) {
#define BS_HY_CPL(II)                                                                                   \
    if (I == II) {                                                                                      \
        if (cpl == 1) return go_hybrid<K, O, W, II, 1>(params, q, m, out, threads, grid, smem, s, uns); \
        if (cpl == 2) return go_hybrid<K, O, W, II, 2>(params, q, m, out, threads, grid, smem, s, uns); \
        if (cpl == 4) return go_hybrid<K, O, W, II, 4>(params, q, m, out, threads, grid, smem, s, uns); \
    }
    if constexpr (W >= 1) BS_HY_CPL(1)
    if constexpr (W >= 2) BS_HY_CPL(2)
    if constexpr (W >= 4) BS_HY_CPL(4)
    if constexpr (W >= 8) BS_HY_CPL(8)
#undef BS_HY_CPL
    *uns = true;
    return cudaSuccess;
}

template <class K, class O>
static cudaError_t dispatch_hybrid(const void* params, const void* q, uint64_t m, void* out, uint32_t threads,
                                   uint32_t W, uint32_t I, uint32_t cpl, Grid grid, uint32_t smem,
                                   cudaStream_t s, bool* uns) {
    switch (W) {
        case 2: return hybrid_w<K, O, 2>(params, q, m, out, threads, I, cpl, grid, smem, s, uns);
        case 4: return hybrid_w<K, O, 4>(params, q, m, out, threads, I, cpl, grid, smem, s, uns);
        case 8: return hybrid_w<K, O, 8>(params, q, m, out, threads, I, cpl, grid, smem, s, uns);
        case 16: return hybrid_w<K, O, 16>(params, q, m, out, threads, I, cpl, grid, smem, s, uns);
        default: *uns = true; return cudaSuccess;
    }
}

cudaError_t launch_kary_hybrid(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                               uint32_t threads, uint32_t W, uint32_t I, uint32_t cpl, Grid grid,
                               uint32_t smem, cudaStream_t s, bool* uns) {
    *uns = false;
    if (kb == 8 && ob == 8) return dispatch_hybrid<uint64_t, uint64_t>(params, q, m, out, threads, W, I, cpl, grid, smem, s, uns);
    if (kb == 8 && ob == 4) return dispatch_hybrid<uint64_t, uint32_t>(params, q, m, out, threads, W, I, cpl, grid, smem, s, uns);
    if (kb == 4 && ob == 8) return dispatch_hybrid<uint32_t, uint64_t>(params, q, m, out, threads, W, I, cpl, grid, smem, s, uns);
    return dispatch_hybrid<uint32_t, uint32_t>(params, q, m, out, threads, W, I, cpl, grid, smem, s, uns);
}

}  // namespace bs
