// kary_g1.cuh — K-ary search (§5), "thread-per-lookup"
// B200 schedule for small nodes (kary_mode 6, and 7 = the bench default).
//
// Same index and result as kary.cu.  Designed around the two limits the
// tiered schedule (kary_tiered.cuh) runs into on B200 — issue slots and L1
// data-pipe wavefronts:
//
//  * FLAT (kary_mode 7): the shared-memory levels are replaced by ONE binary
//    search over a pinned Eytzinger table of the maxima of the nodes of one
//    K-ary level (Index::d_flat) — §4.2's pinned top levels of a binary search
//    feeding §5's K-ary levels; D probes, no per-level bookkeeping.
//  * shared-memory levels: ONE thread per lookup, binary search inside each
//    node over the image's hi-word plane only (u64; u32 keys are exact).  A
//    lane whose query ties a separator's hi word fixes its node by stepping
//    over the level's maxima that share q's hi word and are still < q, read
//    from the sorted array (only the tied lanes, usually one load; at small n
//    a hit query equals a leaf maximum 1 time in C).  With the lo plane out of shared memory, twice as many levels fit.
//  * global separator levels: still ONE thread per lookup — a node of
//    W*key <= 64 B is one or two 256-bit loads (sm_100 LDG.E.ENL2.256) by the
//    owning thread, so a level costs ~17 instructions per 32 lookups and no
//    cross-lane traffic.  Small nodes (K = 5: 32 B, one sector) keep the L2
//    traffic low; the extra levels are cheap because they are per thread.
//  * leaf: GL = C*key/32 lanes per lookup, one 256-bit load each, so a 128-B
//    leaf line is ONE wavefront; (key, chunk) arrive by __shfl_sync from the
//    owner, the count is a packed full-warp REDUX (no wavefront), hit by
//    __ballot_sync, and the group's last lane stores the result (a wave's
//    32/GL results are contiguous).
#pragma once
#include "common.cuh"
#include "kary_tiered.cuh"
#include "params.h"
#include "peer_sync.cuh"

namespace bs {

// n x 32-B vector loads of a node / leaf piece (u64: 4 keys, u32: 8 keys per load)
template <class K, int NV>
__device__ __forceinline__ void ld_node(const K* p, bool hint, uint64_t pol, K* x) {
    constexpr int V32 = 32 / (int)sizeof(K);
    if constexpr (NV * (int)sizeof(K) <= 16) {
        ldv<K, NV>(p, hint, pol, x);
    } else {
#pragma unroll
        for (int t = 0; t < NV / V32; ++t) ldv<K, V32>(p + t * V32, hint, pol, x + t * V32);
    }
}

// Order-preserving 32-bit image of a u64 key for the flat table and its level
// image (KaryParams::fbase / fshift; the hi word when the keys span 2^64, exact
// when they span < 2^32, so keys sharing their hi word do not tie).
__device__ __forceinline__ uint32_t flat_image(uint64_t x, uint64_t base, uint32_t sh) {
    if (x <= base) return 0u;
    const uint64_t d = (x - base) >> sh;
    return d > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)d;
}

// #{slots < q} of one image node (W sorted 32-bit slots) by binary search; `tie`
// records a probe equal to q's image (then the count may be short, fixed later)
template <int W>
__device__ __forceinline__ uint32_t img32_rank(const uint32_t* S, uint32_t nd, uint32_t fq, bool extra, bool& tie) {
    uint32_t c = 0;
#pragma unroll
    for (int s = W / 2; s >= 1; s >>= 1) {
        const uint32_t h = S[nd + c + s - 1];
        tie |= h == fq;
        c += h < fq ? (uint32_t)s : 0u;
    }
    if (extra) {
        const uint32_t h = S[nd + c];
        tie |= h == fq;
        c += h < fq ? 1u : 0u;
    }
    return c;
}

// First node c' >= c whose maximum a[min((c'+1)*span, n) - 1] is >= q, or M:
// the exact node after a descent over images that only bound it from below.
// Galloping then bisection: O(log #tied maxima) reads, never a linear walk.
template <class K>
__device__ __forceinline__ uint64_t step_over_ties(const K* __restrict__ a, uint64_t n, uint64_t span, uint64_t M,
                                                   uint64_t c, K q) {
    auto mx = [&](uint64_t i) -> K {
        uint64_t e = (i + 1) * span;
        if (e > n) e = n;
        return ldg(a + e - 1);
    };
    if (c >= M || mx(c) >= q) return c;
    uint64_t l = c + 1, step = 1, h;
    for (;;) {
        h = l - 1 + step;
        if (h >= M) { h = M; break; }
        if (mx(h) >= q) break;
        l = h + 1;
        step <<= 1;
    }
    while (l < h) {
        const uint64_t mid = l + ((h - l) >> 1);
        if (mx(mid) < q) l = mid + 1;
        else h = mid;
    }
    return l;
}

// OBC != 0: the output width is a compile-time constant (the FLAT T = 1
// instance for out_bytes == key_bytes), so the epilogue carries no width select
template <class K, int W, int GL, int IL, int T, bool FLAT, bool PEER = false, int OBC = 0>
__global__ void __launch_bounds__(T >= 2 ? 768 : 1024, 1)
k_kary_g1(const KaryParams<K> p, const K* __restrict__ q, uint64_t m_arg, void* __restrict__ out, uint32_t ob_arg) {
    const uint32_t ob = OBC ? (uint32_t)OBC : ob_arg;
    constexpr int VL = 32 / (int)sizeof(K);     // leaf keys per lane (one 256-bit load)
    constexpr int GPWL = 32 / GL;               // leaf lookups per wave
    constexpr uint32_t GMASK = (GL == 32) ? 0xFFFFFFFFu : ((1u << GL) - 1u);
    static_assert(GL >= 1 && 32 % GL == 0 && GL % IL == 0, "bad leaf shape");
    static_assert(W * (int)sizeof(K) <= 64, "node of at most two 256-bit loads");

    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.smem_bytes - 16);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t jl = lane % GL;               // lane within its leaf group
    const uint32_t gl = lane / GL;               // leaf group within the warp
    const uint32_t gm = GMASK << (gl * GL);

    if (FLAT) stage_image<uint32_t, false>(S, p.flat, 0, (1u << p.flat_D) + p.flat_img_words, bar);
    else if (p.img_words) stage_image<uint32_t, false>(S, p.img, p.img_plane_words, p.img_words, bar);

    // fused peer routing (bs_lookup_peer): wait until every rank has routed
    // its queries into this rank's window; the slot count is on the device
    constexpr bool peer = PEER;   // PEER instances exist for T = 1 only (go_g1)
    uint64_t m = m_arg;
    if constexpr (PEER) {
        if (threadIdx.x == 0) peer_wait_ge(p.peer_wait, p.peer_wait_target, p.peer_err);
        __syncthreads();
        const uint64_t got = *(volatile const unsigned long long*)p.peer_cursor;
        m = got < m_arg ? got : m_arg;
    }

    // one instruction form per access: the hint knobs select the POLICY
    // (evict_normal when off), so no access is issued twice under opposite
    // predicates (a runtime choice between the hinted and the plain form did)
    const uint64_t pol_normal = policy_evict_normal();
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : pol_normal;
    const uint64_t pol_leaf = p.leaf_hint ? policy_evict_first() : pol_normal;
    const uint64_t pol_sep = p.sep_hint ? policy_evict_last() : pol_normal;
    const uint64_t n = p.n;
    const uint32_t K_ = p.K, C = p.C, L = p.L, Ls = p.Ls;
    const bool extra = (K_ - 1 == (uint32_t)W);
    const uint32_t fb_leaf = bitlen_c(C - 1);
    const uint64_t warps_total = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nwt = (m + 31) / 32;
    uint64_t wt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    auto load_tile = [&](uint64_t t) -> K {
        const uint64_t i = t * 32 + lane;
        if (t >= nwt || i >= m) return KeyMax<K>::v;
        // PEER: the receive window is written by other GPUs while this kernel is
        // resident (before the acquire in peer_wait_ge), so its queries are read
        // with the coherent L2 path (ld.global.cg), never the non-coherent one
        if constexpr (PEER) return __ldcg(q + i);
        else return load_stream(q + i, true, pol_stream);
    };

    // T warp-tiles per iteration: each thread carries T independent lookups
    // through the shared and global levels (T loads in flight per thread)
    const uint64_t wstep = warps_total * T;
    wt = wt * T;
    K key_n[T];
#pragma unroll
    for (int t = 0; t < T; ++t) key_n[t] = load_tile(wt + t);
    for (; wt < nwt; wt += wstep) {
        K key[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            key[t] = key_n[t];
            key_n[t] = load_tile(wt + wstep + t);
        }
        // PEER: each owner lane fetches its slot's return tag now; the load is
        // hidden behind the descent, the leaf epilogue takes it by shuffle
        uint32_t tag_own[T];
        if constexpr (PEER) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const uint64_t i = (wt + t) * 32 + lane;
                tag_own[t] = i < m ? __ldcg(p.peer_tag + i) : 0u;
            }
        }
        // ---- shared-memory levels: hi words only, exact redo on a tie ----
        uint32_t node[T];
        bool tie = false;
#pragma unroll
        for (int t = 0; t < T; ++t) node[t] = 0;
        if constexpr (FLAT) {
            // binary search over the pinned Eytzinger table of level-Ls node maxima:
            // k <- 2k + [T[k] < q] for D levels; the rank k - 2^D is the node
            // The recurrence runs on the shared ADDRESS a = sb + 4k: a' = 2a - sb +
            // 4[T[k] < q] is one SEL + one IMAD per level (no index -> address step).
            // u64 hi-word ties: a table entry on the path equals q's hi word iff the
            // last left-turn node (k >> ffs(~k), the lower-bound entry) does — every
            // left turn below a tied node stays within [qh, qh] — so one probe after
            // the loop replaces a compare per level.
            const uint32_t D = p.flat_D;
            const uint32_t sb = smem_u32(S);
            const uint32_t step_lt = 4u - sb, step_ge = 0u - sb;
            uint32_t a[T], k[T], fq[T];
#pragma unroll
            for (int t = 0; t < T; ++t) {
                a[t] = sb + 4u;
                if constexpr (sizeof(K) == 8) fq[t] = flat_image((uint64_t)key[t], p.fbase, p.fshift);
                else fq[t] = (uint32_t)key[t];
            }
#pragma unroll 4
            for (uint32_t d = 0; d < D; ++d) {
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const uint32_t h = lds_u32(a[t]);
                    a[t] = 2u * a[t] + (h < fq[t] ? step_lt : step_ge);
                }
            }
#pragma unroll
            for (int t = 0; t < T; ++t) {
                k[t] = (a[t] - sb) >> 2;
                node[t] = k[t] - (1u << D);
                if constexpr (sizeof(K) == 8) {
                    const uint32_t j = k[t] >> __ffs(~k[t]);
                    tie |= j != 0 && S[j] == fq[t];
                }
            }
            if (p.flat_img_words) {
                // one more shared level: the flat level's node image follows the table
                const uint32_t last = p.nodes_next[Ls - 1] - 1;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const uint32_t c = img32_rank<W>(S, (1u << D) + node[t] * (W + 1), fq[t], extra, tie);
                    const uint32_t child = node[t] * K_ + c;
                    node[t] = child < last ? child : last;
                }
            }
            if constexpr (sizeof(K) == 8) {
                // image ties: node = #(maxima whose image < q's), a lower bound on
                // the exact count; the tied lanes step over the maxima that are
                // still < q — read from the sorted array (max of node c =
                // a[min((c+1)*span, n) - 1]), galloping: usually one read
                if (__any_sync(0xFFFFFFFFu, tie) && tie) {
#pragma unroll 1
                    for (int t = 0; t < T; ++t)
                        node[t] = (uint32_t)step_over_ties(p.a, n, p.flat_span, p.flat_M, node[t], key[t]);
                }
            }
        } else {
        for (uint32_t l = 0; l < Ls; ++l) {
            const uint32_t last = p.nodes_next[l] - 1;
            const uint32_t base = p.img_base[l];
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const uint32_t c = smem_node_rank<K, W, false, false>(S, base + node[t] * (W + 1), key[t], extra, tie);
                const uint32_t child = node[t] * K_ + c;
                node[t] = child < last ? child : last;
            }
        }
        if constexpr (sizeof(K) == 8) {
            // a hi-word tie (q equals a separator's top half: ~1 in C per lookup
            // at the leaf-max level of a small index) is fixed by the tied lanes
            // (the hi-word descent is exact for the hi-word order, so node is
            // #(level-Ls subtree maxima whose hi word < q's): step the tied
            // lanes over the maxima that share q's hi word and are still < q,
            // read from the sorted array — usually one load)
            if (__any_sync(0xFFFFFFFFu, tie) && tie) {
#pragma unroll 1
                for (int t = 0; t < T; ++t)
                    node[t] = (uint32_t)step_over_ties(p.a, n, p.flat_span, p.flat_M, node[t], key[t]);
            }
        }
        }
        // ---- global separator levels: thread per lookup, whole node in registers ----
        for (uint32_t l = Ls; l < L; ++l) {
            const K* lv = p.sep + p.lvl_base[l];
            const uint32_t last = p.nodes_next[l] - 1;
            K s[T][W];
            // evict_last only for the levels that fit L2 (cumulative); deeper ones stream like leaves
            const uint64_t pol_l = l < p.sep_last_end ? pol_sep : pol_leaf;
#pragma unroll
            for (int t = 0; t < T; ++t) ld_node<K, W>(lv + (uint64_t)node[t] * W, true, pol_l, s[t]);
#pragma unroll
            for (int t = 0; t < T; ++t) {
                uint32_t c = 0;
#pragma unroll
                for (int v = 0; v < W; ++v) c += (s[t][v] < key[t]) ? 1u : 0u;
                const uint32_t child = node[t] * K_ + c;
                node[t] = child < last ? child : last;
            }
        }
        // ---- leaf: GL lanes per lookup, IL waves in flight, T tiles ----
#pragma unroll
        for (int t = 0; t < T; ++t) {
#pragma unroll 1
        for (int b = 0; b < GL / IL; ++b) {
            K kk[IL];
            uint32_t cc[IL];
            K x[IL][VL];
#pragma unroll
            for (int i = 0; i < IL; ++i) {
                const int src = (b * IL + i) * GPWL + (int)gl;
                kk[i] = __shfl_sync(0xFFFFFFFFu, key[t], src);
                cc[i] = __shfl_sync(0xFFFFFFFFu, node[t], src);
                ldv<K, VL>(p.a + (uint64_t)cc[i] * C + jl * VL, true, pol_leaf, x[i]);
            }
#pragma unroll
            for (int i = 0; i < IL; ++i) {
                // MAX padding past n never counts and cannot make a hit (lb == n);
                // the chunk's last key (last lane) is added back after the packed sum
                uint32_t lt = 0;
                bool eq = false;
#pragma unroll
                for (int u = 0; u < VL; ++u) {
                    if (u < VL - 1 || jl != GL - 1) lt += (x[i][u] < kk[i]) ? 1u : 0u;
                    eq |= x[i][u] == kk[i];
                }
                const bool last_lt = x[i][VL - 1] < kk[i];
                lt = group_sum<GL>(lt, gl, fb_leaf);
                const bool any_eq = (__ballot_sync(0xFFFFFFFFu, eq) & gm) != 0;
                uint32_t tg = 0;
                if constexpr (PEER) tg = __shfl_sync(0xFFFFFFFFu, tag_own[t], (b * IL + i) * GPWL + (int)gl);
                if (jl == GL - 1) {
                    const uint64_t lbv = (uint64_t)cc[i] * C + lt + (last_lt ? 1u : 0u);
                    const bool hit = any_eq && lbv < n;
                    const uint64_t miss = ob == 8 ? (1ull << 63) : (1ull << 31);
                    const uint64_t res = hit ? lbv : (lbv | miss);
                    const uint64_t o = (wt + t) * 32 + (uint64_t)((b * IL + i) * GPWL) + gl;
                    if (o < m) {
                        if constexpr (PEER) {
                            // result straight into the source rank's return window (P2P store)
                            const uint64_t g = lbv + p.peer_base;
                            // 4-B tag: rank in the top bits (u64 shift: peer_shift = 32 at P = 1)
                            const uint32_t sh = p.peer_shift;
                            p.peer_ret[(uint64_t)tg >> sh][tg & (uint32_t)((1ull << sh) - 1ull)] = hit ? g : (g | miss);
                        } else if (ob == 8) {
                            store_stream((uint64_t*)out + o, res, true, pol_stream);
                        } else {
                            store_stream((uint32_t*)out + o, (uint32_t)res, true, pol_stream);
                        }
                    }
                }
            }
        }
        }
    }
    if (PEER && peer_last_cta(p.peer_done)) {
        // every CTA has read the cursor (at its start) and stored its results:
        // re-arm the window, then tell every rank its results have landed
        *p.peer_cursor = 0;
        __threadfence_system();
        for (uint32_t r = 0; r < p.peer_P; ++r) red_release_sys_add_u64(p.peer_sig[r], 1ull);
    }
}

// PIPE variant of the FLAT schedule (T = 1): the D probes of the NEXT
// warp-tile's pinned-table search are spread over this tile's load stages
// (global levels + leaf), so the shared-memory search costs issue slots but
// never exposes its latency; the warp always has global loads in flight.
template <class K, int W, int GL, int IL>
__global__ void __launch_bounds__(1024, 1)
k_kary_g1p(const KaryParams<K> p, const K* __restrict__ q, uint64_t m, void* __restrict__ out, uint32_t ob) {
    constexpr int VL = 32 / (int)sizeof(K);
    constexpr int GPWL = 32 / GL;
    constexpr uint32_t GMASK = (GL == 32) ? 0xFFFFFFFFu : ((1u << GL) - 1u);
    static_assert(GL >= 1 && 32 % GL == 0 && GL % IL == 0, "bad leaf shape");

    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.smem_bytes - 16);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t jl = lane % GL;
    const uint32_t gl = lane / GL;
    const uint32_t gm = GMASK << (gl * GL);

    stage_image<uint32_t, false>(S, p.flat, 0, 1u << p.flat_D, bar);

    // one instruction form per access: the hint knobs select the POLICY
    // (evict_normal when off), so no access is issued twice under opposite
    // predicates (a runtime choice between the hinted and the plain form did)
    const uint64_t pol_normal = policy_evict_normal();
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : pol_normal;
    const uint64_t pol_leaf = p.leaf_hint ? policy_evict_first() : pol_normal;
    const uint64_t pol_sep = p.sep_hint ? policy_evict_last() : pol_normal;
    const uint64_t n = p.n;
    const uint32_t K_ = p.K, C = p.C, L = p.L, Ls = p.Ls, D = p.flat_D;
    const uint32_t fb_leaf = bitlen_c(C - 1);
    const uint32_t stages = (L - Ls) + 1;
    const uint32_t per = (D + stages - 1) / stages;   // probes of the next tile per load stage
    const uint64_t warps_total = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nwt = (m + 31) / 32;
    uint64_t wt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    auto load_tile = [&](uint64_t t) -> K {
        const uint64_t i = t * 32 + lane;
        return (t < nwt && i < m) ? load_stream(q + i, true, pol_stream) : KeyMax<K>::v;
    };
    auto probe = [&](uint32_t& k, K kq, bool& tie) {
        const uint32_t h = S[k];
        bool less;
        if constexpr (sizeof(K) == 8) {
            const uint32_t qh = flat_image((uint64_t)kq, p.fbase, p.fshift);
            less = h < qh;
            tie |= h == qh;
        } else {
            less = h < (uint32_t)kq;
        }
        k = 2 * k + (less ? 1u : 0u);
    };
    auto exact = [&](K kq) -> uint32_t {
        uint32_t k = 1;
        for (uint32_t d = 0; d < D; ++d) k = 2 * k + ((ldg(p.flat64 + k) < (uint64_t)kq) ? 1u : 0u);
        return k;
    };

    K key = load_tile(wt);
    uint32_t node;
    {
        uint32_t k = 1;
        bool tie = false;
        for (uint32_t d = 0; d < D; ++d) probe(k, key, tie);
        if constexpr (sizeof(K) == 8) {
            if (__any_sync(0xFFFFFFFFu, tie)) k = exact(key);
        }
        node = k - (1u << D);
    }
    K key_n = load_tile(wt + warps_total);
    K knext = load_tile(wt + 2 * warps_total);

    for (; wt < nwt; wt += warps_total) {
        uint32_t kn = 1, dn = 0;
        bool tie_n = false;
        // ---- global separator levels of tile t, next tile's probes in between ----
        for (uint32_t l = Ls; l < L; ++l) {
            K s[W];
            // evict_last only for the levels that fit L2 (as k_kary_g1)
            ld_node<K, W>(p.sep + p.lvl_base[l] + (uint64_t)node * W, true, l < p.sep_last_end ? pol_sep : pol_leaf, s);
            for (uint32_t r = 0; r < per && dn < D; ++r, ++dn) probe(kn, key_n, tie_n);
            uint32_t c = 0;
#pragma unroll
            for (int v = 0; v < W; ++v) c += (s[v] < key) ? 1u : 0u;
            const uint32_t child = node * K_ + c;
            const uint32_t last = p.nodes_next[l] - 1;
            node = child < last ? child : last;
        }
        // ---- leaf of tile t ----
#pragma unroll 1
        for (int b = 0; b < GL / IL; ++b) {
            K kk[IL];
            uint32_t cc[IL];
            K x[IL][VL];
#pragma unroll
            for (int i = 0; i < IL; ++i) {
                const int src = (b * IL + i) * GPWL + (int)gl;
                kk[i] = __shfl_sync(0xFFFFFFFFu, key, src);
                cc[i] = __shfl_sync(0xFFFFFFFFu, node, src);
                ldv<K, VL>(p.a + (uint64_t)cc[i] * C + jl * VL, true, pol_leaf, x[i]);
            }
            for (; dn < D; ++dn) probe(kn, key_n, tie_n);
#pragma unroll
            for (int i = 0; i < IL; ++i) {
                uint32_t lt = 0;
                bool eq = false;
#pragma unroll
                for (int u = 0; u < VL; ++u) {
                    if (u < VL - 1 || jl != GL - 1) lt += (x[i][u] < kk[i]) ? 1u : 0u;
                    eq |= x[i][u] == kk[i];
                }
                const bool last_lt = x[i][VL - 1] < kk[i];
                lt = group_sum<GL>(lt, gl, fb_leaf);
                const bool any_eq = (__ballot_sync(0xFFFFFFFFu, eq) & gm) != 0;
                if (jl == GL - 1) {
                    const uint64_t lbv = (uint64_t)cc[i] * C + lt + (last_lt ? 1u : 0u);
                    const bool hit = any_eq && lbv < n;
                    const uint64_t miss = ob == 8 ? (1ull << 63) : (1ull << 31);
                    const uint64_t res = hit ? lbv : (lbv | miss);
                    const uint64_t o = wt * 32 + (uint64_t)((b * IL + i) * GPWL) + gl;
                    if (o < m) {
                        if (ob == 8) store_stream((uint64_t*)out + o, res, true, pol_stream);
                        else store_stream((uint32_t*)out + o, (uint32_t)res, true, pol_stream);
                    }
                }
            }
        }
        if constexpr (sizeof(K) == 8) {
            if (__any_sync(0xFFFFFFFFu, tie_n)) kn = exact(key_n);
        }
        node = kn - (1u << D);
        key = key_n;
        key_n = knext;
        knext = load_tile(wt + 3 * warps_total);
    }
}

template <class K, int W, int GL, int IL>
static cudaError_t go_g1(const void* params, const void* q, uint64_t m, void* out, uint32_t ob, uint32_t threads,
                         uint32_t T, bool flat, Grid grid, uint32_t smem, cudaStream_t s, bool* uns) {
    // bs_lookup_peer fills the peer fields: the PEER instance (T = 1) carries the epilogue
    const bool peer = ((const KaryParams<K>*)params)->peer_cursor != nullptr;
    auto kern = flat ? (T >= 2 ? k_kary_g1<K, W, GL, IL, 2, true> : k_kary_g1<K, W, GL, IL, 1, true>)
                     : (T >= 2 ? k_kary_g1<K, W, GL, IL, 2, false> : k_kary_g1<K, W, GL, IL, 1, false>);
    if (peer) kern = flat ? k_kary_g1<K, W, GL, IL, 1, true, true> : k_kary_g1<K, W, GL, IL, 1, false, true>;
    // BS_G1_RUNTIME_OB=1 keeps the runtime-width instance (A/B knob, not part of the ABI)
    static const bool runtime_ob = getenv("BS_G1_RUNTIME_OB") != nullptr;
    if (flat && T == 1 && !peer && ob == sizeof(K) && !runtime_ob)
        kern = k_kary_g1<K, W, GL, IL, 1, true, false, (int)sizeof(K)>;
    if (flat && T == 3 && !peer) kern = k_kary_g1p<K, W, GL, IL>;   // T = 3 encodes "pipelined, one lookup per thread"
    const uint64_t need = (m + threads - 1) / threads;
    uint64_t g = 0;
    cudaError_t e = plan_grid((const void*)kern, threads, smem, grid, need, carveout_for(smem, threads), &g, uns);
    if (e != cudaSuccess || *uns) return e;
    kern<<<(unsigned)g, threads, smem, s>>>(*(const KaryParams<K>*)params, (const K*)q, m, out, ob);
    count_launch();
    return cudaGetLastError();
}

// W = node slots (W*key <= 64 B), GL = leaf lanes (C*key = 32*GL), IL = leaf waves in flight
template <class K>
cudaError_t dispatch_g1(const void* params, const void* q, uint64_t m, void* out, uint32_t ob, uint32_t threads,
                        uint32_t W, uint32_t GL, uint32_t IL, uint32_t T, bool flat, Grid grid, uint32_t smem,
                        cudaStream_t s, bool* uns) {
#define BS_G1_IL(WW, GG)                                                                                  \
    {                                                                                                     \
        if (IL >= 4 && GG >= 4) return go_g1<K, WW, GG, (GG >= 4 ? 4 : 1)>(params, q, m, out, ob, threads, T, flat, grid, smem, s, uns); \
        if (IL >= 2 && GG >= 2) return go_g1<K, WW, GG, (GG >= 2 ? 2 : 1)>(params, q, m, out, ob, threads, T, flat, grid, smem, s, uns); \
        return go_g1<K, WW, GG, 1>(params, q, m, out, ob, threads, T, flat, grid, smem, s, uns);                  \
    }
#define BS_G1_G(WW)                             \
    case WW:                                    \
        if (GL == 1) BS_G1_IL(WW, 1)            \
        if (GL == 2) BS_G1_IL(WW, 2)            \
        if (GL == 4) BS_G1_IL(WW, 4)            \
        if (GL == 8) BS_G1_IL(WW, 8)            \
        break;
    constexpr int WMAX = 64 / (int)sizeof(K);
    switch (W) {
        BS_G1_G(2)
        BS_G1_G(4)
        BS_G1_G(8)
        case 16:
            if constexpr (WMAX >= 16) {
                if (GL == 1) BS_G1_IL(16, 1)
                if (GL == 2) BS_G1_IL(16, 2)
                if (GL == 4) BS_G1_IL(16, 4)
                if (GL == 8) BS_G1_IL(16, 8)
            }
            break;
        default: break;
    }
#undef BS_G1_G
#undef BS_G1_IL
    *uns = true;
    return cudaSuccess;
}

}  // namespace bs
