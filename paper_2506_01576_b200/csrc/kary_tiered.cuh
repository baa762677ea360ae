// kary_tiered.cuh — K-ary search (§5), "tiered" B200 schedule.
//
// Same index as kary.cu (chunk-max separators, top-first levels of W-slot
// nodes, child m*K+j, leaf = the unpermuted sorted array; reading R16) and the
// same result word.  Each tier of the memory hierarchy gets the schedule that
// is cheapest there:
//
//  * shared-memory levels (the top Ls levels, staged once per CTA by TMA: the
//    §5.1 "pinning" of KS): ONE thread per lookup, and the thread finds
//    its child with a branch-free binary search inside the node
//    (log2(W) dependent 8-B shared loads, +1 when K-1 == W) instead of reading
//    all W slots — a node is sorted, so this is the same count of separators
//    < q at a quarter of the shared-memory wavefronts.
//  * global levels + leaf (L2 / HBM): G = W*key/16 lanes per lookup, each lane
//    one 16-B vector load, so a node is ONE coalesced request of W*key bytes
//    ("K-1 threads compare in parallel"; on B200 one 128-B line for
//    K = 17 u64).  The group counts separators < q with one __ballot_sync per
//    vector element and __popc.  A warp's 32 lookups are handed to its 32/G
//    groups in G waves (__shfl_sync), I waves in flight at a time.
//  * leaf: CPL = C/G keys per lane (R = C/W vector loads of 16 B); positions
//    >= n read the MAX padding that bs_build writes and are masked out.
//  * each group's first lane stores its result (a wave's 32/G results are
//    contiguous); the next warp-tile's queries are prefetched during the descent.
#pragma once
#include "common.cuh"
#include "params.h"

namespace bs {

// V keys (V*sizeof(K) in {8, 16} bytes) from global memory, no L1 allocation,
// optional L2 eviction-priority policy.
template <class K, int V>
__device__ __forceinline__ void ldv(const K* p, bool hint, uint64_t pol, K* x) {
    if constexpr (sizeof(K) == 8) {
        static_assert(V == 2, "u64: 16-B vectors");
        if (hint)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                         : "=l"(x[0]), "=l"(x[1]) : "l"(p), "l"(pol));
        else
            asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(x[0]), "=l"(x[1]) : "l"(p));
    } else if constexpr (V == 4) {
        if (hint)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                         : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "l"(p), "l"(pol));
        else
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "l"(p));
    } else {
        static_assert(V == 2, "u32: 8- or 16-B vectors");
        if (hint)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                         : "=r"(x[0]), "=r"(x[1]) : "l"(p), "l"(pol));
        else
            asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(x[0]), "=r"(x[1]) : "l"(p));
    }
}

// slot < key for a slot of the shared-memory image: u32 keys read the one
// plane; u64 keys read the hi-word plane and, only when the hi words tie, the
// lo-word plane (one 4-B bank access per probe).
// The lo plane sits at a fixed shared-memory offset so its probe is the hi
// probe's address plus an immediate.
constexpr uint32_t kImgLoWords = 29056;   // 116224 B = half of sm_100's 227 KB opt-in

template <class K, bool PAIR>
__device__ __forceinline__ bool img_less(const uint32_t* S, uint32_t w, K key) {
    if constexpr (PAIR) {
        return reinterpret_cast<const uint64_t*>(S)[w] < (uint64_t)key;
    } else if constexpr (sizeof(K) == 8) {
        const uint32_t qh = (uint32_t)((uint64_t)key >> 32);
        const uint32_t h = S[w];
        bool less = h < qh;
        if (h == qh) less = S[kImgLoWords + w] < (uint32_t)key;
        return less;
    } else {
        return S[w] < (uint32_t)key;
    }
}

// #{slots < key} of one shared-memory node (W sorted slots, MAX-padded past
// K-1), by branch-free binary search over the image; `extra` = (K-1 == W)
// adds the final compare that distinguishes "all W < key".
template <class K, int W, bool PAIR>
__device__ __forceinline__ uint32_t smem_node_rank(const uint32_t* S, uint32_t nd, K key, bool extra) {
    uint32_t c = 0;
#pragma unroll
    for (int s = W / 2; s >= 1; s >>= 1) c += img_less<K, PAIR>(S, nd + c + s - 1, key) ? (uint32_t)s : 0u;
    if (extra) c += img_less<K, PAIR>(S, nd + c, key) ? 1u : 0u;
    return c;
}

// Stage the first `words` words of each image plane with TMA bulk copies:
// hi (or the u32 plane) at word 0, lo at word kImgLoWords.
template <class K, bool PAIR>
__device__ __forceinline__ void stage_image(uint32_t* S, const uint32_t* img, uint64_t plane_words, uint32_t words,
                                            uint64_t* bar) {
    constexpr uint32_t planes = (sizeof(K) == 8 && !PAIR) ? 2 : 1;
    constexpr uint32_t unit = PAIR ? 8 : 4;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, words * unit * planes);
        constexpr uint32_t CH = 32768;
        for (uint32_t pl = 0; pl < planes; ++pl)
            for (uint32_t o = 0; o < words * unit; o += CH) {
                const uint32_t b = (words * unit - o < CH) ? (words * unit - o) : CH;
                bulk_g2s((char*)(S + pl * kImgLoWords) + o, (const char*)(img + pl * plane_words) + o, b, bar);
            }
    }
    mbar_wait(bar, 0);
}

template <class K, int W, int R, int I, bool PAIR>
__global__ void __launch_bounds__(1024, 1)
k_kary_tiered(const KaryParams<K> p, const K* __restrict__ q, uint64_t m, void* __restrict__ out, uint32_t ob) {
    constexpr int V = (16 / (int)sizeof(K)) < W ? (16 / (int)sizeof(K)) : W;   // keys per lane per load
    constexpr int G = W / V;                                                  // lanes per lookup
    constexpr int GPW = 32 / G;                                               // lookups per wave
    constexpr int CPL = R * V;                                                // leaf keys per lane
    constexpr uint32_t GMASK = (G == 32) ? 0xFFFFFFFFu : ((1u << G) - 1u);
    static_assert(G >= 1 && 32 % G == 0 && G % I == 0, "bad tiered shape");

    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.smem_bytes - 16);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t j = lane % G;              // my lane within my group
    const uint32_t g = lane / G;              // my group within the warp
    const uint32_t gm = GMASK << (g * G);     // my group's lanes in a ballot

    if (p.img_words) stage_image<K, PAIR>(S, p.img, p.img_plane_words, p.img_words, bar);

    const uint64_t pol_first = policy_evict_first();
    const uint64_t pol_last = policy_evict_last();
    const bool sh = p.stream_hint != 0, lh = p.leaf_hint != 0, sep_last = p.sep_hint != 0;
    const uint64_t n = p.n;
    const uint32_t K_ = p.K, C = p.C, L = p.L, Ls = p.Ls;
    const bool extra = (K_ - 1 == (uint32_t)W);
    const uint64_t warps_total = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nwt = (m + 31) / 32;
    uint64_t wt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    // One shared-memory level of the thread-per-lookup descent.
    auto smem_level = [&](uint32_t l, K key, uint32_t node) -> uint32_t {
        const uint32_t c = smem_node_rank<K, W, PAIR>(S, p.img_base[l] + node * (W + 1), key, extra);
        const uint32_t child = node * K_ + c;
        const uint32_t last = p.nodes_next[l] - 1;
        return child < last ? child : last;
    };
    auto load_tile = [&](uint64_t t) -> K {
        const uint64_t i = t * 32 + lane;
        return (t < nwt && i < m) ? load_stream(q + i, sh, pol_first) : KeyMax<K>::v;
    };

    // Software pipeline across warp-tiles: while the groups of this warp wait
    // on the global-level and leaf loads of tile t, all 32 lanes advance the
    // shared-memory descent of tile t+1 one level per load stage, so the
    // shared-memory phase costs issue slots but no exposed latency.
    // key/node: tile t (shared levels done); key_n/node_n: tile t+1 (descending);
    // knext: the queries of tile t+2 (in flight).
    K key = load_tile(wt);
    uint32_t node = 0;
    for (uint32_t l = 0; l < Ls; ++l) node = smem_level(l, key, node);
    K key_n = load_tile(wt + warps_total);
    K knext = load_tile(wt + 2 * warps_total);

    for (; wt < nwt; wt += warps_total) {
        uint32_t node_n = 0, lvl_n = 0;
#pragma unroll 1
        for (int b = 0; b < G / I; ++b) {
            K kk[I];
            uint32_t nn[I];
#pragma unroll
            for (int i = 0; i < I; ++i) {
                const int src = (b * I + i) * GPW + (int)g;
                kk[i] = __shfl_sync(0xFFFFFFFFu, key, src);
                nn[i] = __shfl_sync(0xFFFFFFFFu, node, src);
            }
            for (uint32_t l = Ls; l < L; ++l) {
                const K* lv = p.sep + p.lvl_base[l] + j * V;
                K s[I][V];
#pragma unroll
                for (int i = 0; i < I; ++i) ldv<K, V>(lv + (uint64_t)nn[i] * W, sep_last, pol_last, s[i]);
                if (lvl_n < Ls) { node_n = smem_level(lvl_n, key_n, node_n); ++lvl_n; }
                const uint32_t last = p.nodes_next[l] - 1;
#pragma unroll
                for (int i = 0; i < I; ++i) {
                    uint32_t c = 0;
#pragma unroll
                    for (int v = 0; v < V; ++v) c += __popc(__ballot_sync(0xFFFFFFFFu, s[i][v] < kk[i]) & gm);
                    const uint32_t child = nn[i] * K_ + c;
                    nn[i] = child < last ? child : last;
                }
            }
            // leaf chunk c: lane j holds keys [c*C + j*CPL, +CPL) (MAX-padded past n)
            K x[I][CPL];
#pragma unroll
            for (int i = 0; i < I; ++i) {
                const K* lp = p.a + (uint64_t)nn[i] * C + j * CPL;
#pragma unroll
                for (int t = 0; t < R; ++t) ldv<K, V>(lp + t * V, lh, pol_first, &x[i][t * V]);
            }
            if (lvl_n < Ls) { node_n = smem_level(lvl_n, key_n, node_n); ++lvl_n; }
#pragma unroll
            for (int i = 0; i < I; ++i) {
                // the MAX padding past n is never < q, so it never counts; it can
                // equal q only when q == MAX, and then lb == n (a miss) — hence
                // "hit" also requires lb < n and no per-key bounds test is needed
                uint32_t lt = 0;
                bool eq = false;
#pragma unroll
                for (int t = 0; t < CPL; ++t) {
                    lt += (x[i][t] < kk[i]) ? 1u : 0u;
                    eq |= x[i][t] == kk[i];
                }
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) lt += __shfl_xor_sync(0xFFFFFFFFu, lt, o);
                const uint64_t lbv = (uint64_t)nn[i] * C + lt;
                const bool hit = ((__ballot_sync(0xFFFFFFFFu, eq) & gm) != 0) && lbv < n;
                const uint64_t miss = ob == 8 ? (1ull << 63) : (1ull << 31);
                const uint64_t res = hit ? lbv : (lbv | miss);
                // the group's first lane stores; a wave's GPW results are contiguous
                const uint64_t o = wt * 32 + (uint64_t)((b * I + i) * GPW) + g;
                if (j == 0 && o < m) {
                    if (ob == 8) store_stream((uint64_t*)out + o, res, sh, pol_first);
                    else store_stream((uint32_t*)out + o, (uint32_t)res, sh, pol_first);
                }
            }
        }
        // the rest of tile t+1's shared-memory levels (when they outnumber the load stages)
        for (; lvl_n < Ls; ++lvl_n) node_n = smem_level(lvl_n, key_n, node_n);
        key = key_n;
        node = node_n;
        key_n = knext;
        knext = load_tile(wt + 3 * warps_total);
    }
}

template <class K, int W, int R, int I>
static cudaError_t go_tiered(const void* params, const void* q, uint64_t m, void* out, uint32_t ob, uint32_t threads,
                             bool pair64, Grid grid, uint32_t smem, cudaStream_t s, bool* uns) {
    auto kern = k_kary_tiered<K, W, R, I, false>;
    if constexpr (sizeof(K) == 8) {
        if (pair64) kern = k_kary_tiered<K, W, R, I, true>;
    }
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    if ((int)threads > fa.maxThreadsPerBlock || threads % 32) { *uns = true; return cudaSuccess; }
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint64_t per_cta = (uint64_t)threads;   // one lookup per thread per warp-tile
    const uint64_t need = (m + per_cta - 1) / per_cta;
    uint64_t g = need;
    if (grid.sched_static) {
        int occ = (int)grid.ctas_per_sm;
        if (occ == 0) {
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (int)threads, smem);
            if (e != cudaSuccess) return e;
        }
        if (occ < 1) { *uns = true; return cudaSuccess; }
        g = (uint64_t)grid.sm_count * (uint64_t)occ;
    }
    if (g > need) g = need;
    if (g == 0) g = 1;
    if (g > 0x7FFFFFFFull) g = 0x7FFFFFFFull;
    kern<<<(unsigned)g, threads, smem, s>>>(*(const KaryParams<K>*)params, (const K*)q, m, out, ob);
    return cudaGetLastError();
}

// W = node slots, R = C / W (1, 2, 4), I = waves in flight (clamped to a divisor of G)
template <class K>
cudaError_t dispatch_tiered(const void* params, const void* q, uint64_t m, void* out, uint32_t ob, uint32_t threads,
                            uint32_t W, uint32_t R, uint32_t I, bool pair64, Grid grid, uint32_t smem, cudaStream_t s,
                            bool* uns) {
    constexpr int VK = 16 / (int)sizeof(K);
#define BS_TI_I(WW, RR)                                                                                         \
    {                                                                                                           \
        constexpr int GG = WW / (VK < WW ? VK : WW);                                                            \
        if (GG == 1 || I <= 1) return go_tiered<K, WW, RR, 1>(params, q, m, out, ob, threads, pair64, grid, smem, s, uns); \
        if constexpr (GG >= 4) {                                                                                \
            if (I >= 4) return go_tiered<K, WW, RR, 4>(params, q, m, out, ob, threads, pair64, grid, smem, s, uns);    \
        }                                                                                                       \
        if constexpr (GG >= 2) return go_tiered<K, WW, RR, 2>(params, q, m, out, ob, threads, pair64, grid, smem, s, uns); \
    }
#define BS_TI_R(WW)                          \
    case WW:                                 \
        if (R == 1) BS_TI_I(WW, 1)           \
        if (R == 2) BS_TI_I(WW, 2)           \
        if (R == 4) BS_TI_I(WW, 4)           \
        break;
    switch (W) {
        BS_TI_R(2)
        BS_TI_R(4)
        BS_TI_R(8)
        BS_TI_R(16)
        BS_TI_R(32)
        default: break;
    }
#undef BS_TI_R
#undef BS_TI_I
    *uns = true;
    return cudaSuccess;
}

}  // namespace bs
