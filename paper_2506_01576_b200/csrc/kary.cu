// kary.cu — K-ary search (§5), warp-cooperative on sm_100a.
//
// Layout (built by bs_build, DESIGN.md §"K-ary layout", reading R16): leaf
// chunk c = keys [c*C, (c+1)*C) of the UNPERMUTED sorted array ("the
// leaf layer is the initial sorted array"); separator levels stored top-first,
// each node W = pow2 >= K-1 slots wide (one 128-B line at W*key = 128),
// slot j < K-1 = max key of child m*K+j (MAX past the end and in pad slots);
// child index = m*K + j, no pointers ("we do not need to store child
// pointers").
//
// Search: a group of W lanes owns one lookup; lane j loads slot j of the
// current node (one coalesced line per group), the group counts
// separators < q with __ballot_sync + __popc ("K-1 threads compare in
// parallel ... communicate their results"), which is the child index j of the
// first separator >= q.  32/W lookups per warp-wave, R waves interleaved so R
// independent node loads are in flight per lane.  The leaf chunk is read by
// the same group (C/W keys per lane) and lb = c*C + #keys < q, hit = any key == q.
// Top Ls levels can be staged once per CTA in shared memory (the "pinning"
// optimisation applied to KS, §5.1).
#include "common.cuh"
#include "params.h"

namespace bs {

template <class K, class O, int W, int R>
__global__ void k_kary(const KaryParams<K> p, const K* __restrict__ q, uint64_t m, O* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    K* S = reinterpret_cast<K*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.smem_bytes);
    constexpr int GPW = 32 / W;                 // lookups per warp-wave
    constexpr uint32_t GMASK = (W == 32) ? 0xFFFFFFFFu : ((1u << W) - 1u);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t j = lane & (W - 1);          // slot this lane compares
    const uint32_t g = lane / W;                // group within the warp
    const uint32_t gshift = g * W;

    if (p.smem_bytes) stage_to_smem(S, p.sep, p.smem_bytes, bar);

    const uint64_t pol_first = policy_evict_first();
    const uint64_t pol_last = policy_evict_last();
    const bool sh = p.stream_hint != 0, lh = p.leaf_hint != 0, sep_last = p.sep_hint != 0;
    const uint64_t n = p.n;
    const uint32_t K_ = p.K, C = p.C;
    const uint64_t warps_total = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    constexpr uint32_t PER_WARP = GPW * R;
    const uint64_t nwt = (m + PER_WARP - 1) / PER_WARP;
    uint64_t wt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    // software pipeline: the queries of the next warp-tile are loaded while
    // the current one descends (removes one DRAM round trip per lookup)
    K knext[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint64_t i = wt * PER_WARP + (uint64_t)r * GPW + g;
        knext[r] = (wt < nwt && i < m) ? load_stream(q + i, sh, pol_first) : KeyMax<K>::v;
    }
    for (; wt < nwt; wt += warps_total) {
        const uint64_t base = wt * PER_WARP;
        K key[R];
        uint32_t node[R];
#pragma unroll
        for (int r = 0; r < R; ++r) { key[r] = knext[r]; node[r] = 0; }
        {
            const uint64_t wn = wt + warps_total;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t i = wn * PER_WARP + (uint64_t)r * GPW + g;
                knext[r] = (wn < nwt && i < m) ? load_stream(q + i, sh, pol_first) : KeyMax<K>::v;
            }
        }
        // ---- internal levels: one node per group per level ----
        for (uint32_t l = 0; l < p.L; ++l) {
            K s[R];
            const uint64_t lb = p.lvl_base[l];
            if (l < p.Ls) {
#pragma unroll
                for (int r = 0; r < R; ++r) s[r] = S[lb + (uint64_t)node[r] * W + j];
            } else if (sep_last) {
#pragma unroll
                for (int r = 0; r < R; ++r) s[r] = ld_na_hint(p.sep + lb + (uint64_t)node[r] * W + j, pol_last);
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) s[r] = ld_na(p.sep + lb + (uint64_t)node[r] * W + j);
            }
            const uint32_t last = p.nodes_next[l] - 1;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, s[r] < key[r]);
                const uint32_t cnt = __popc((bal >> gshift) & GMASK);   // first j with q <= sep_j
                const uint32_t child = node[r] * K_ + cnt;
                node[r] = child < last ? child : last;   // children past the end hold no key >= q
            }
        }
        // ---- leaf chunk: lb = c*C + #{keys < q}, hit = any key == q ----
        uint32_t acc[R];   // (count << 1) | hit
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0;
        for (uint32_t t0 = 0; t0 < C; t0 += W) {
            K x[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t pos = (uint64_t)node[r] * C + t0 + j;
                const bool ok = (t0 + j < C) && (pos < n);
                x[r] = ok ? load_key(p.a + pos, lh, pol_first) : KeyMax<K>::v;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t pos = (uint64_t)node[r] * C + t0 + j;
                const bool ok = (t0 + j < C) && (pos < n);
                const uint32_t lt = __ballot_sync(0xFFFFFFFFu, ok && x[r] < key[r]);
                const uint32_t eq = __ballot_sync(0xFFFFFFFFu, ok && x[r] == key[r]);
                acc[r] += (uint32_t)__popc((lt >> gshift) & GMASK) << 1;
                acc[r] |= ((eq >> gshift) & GMASK) ? 1u : 0u;
            }
        }
        if (j == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t i = base + (uint64_t)r * GPW + g;
                if (i < m) {
                    uint64_t lbv = (uint64_t)node[r] * C + (acc[r] >> 1);
                    if (lbv > n) lbv = n;
                    constexpr uint64_t MISS = 1ull << (8 * sizeof(O) - 1);
                    const O res = (O)((acc[r] & 1u) ? lbv : (lbv | MISS));
                    store_stream(out + i, res, sh, pol_first);
                }
            }
        }
    }
}

template <class K, class O, int W, int R>
static cudaError_t go_kary(const void* params, const void* q, uint64_t m, void* out, uint32_t threads,
                           Grid grid, uint32_t smem, cudaStream_t s, bool* uns) {
    auto kern = k_kary<K, O, W, R>;
    const uint64_t per_cta = (uint64_t)(threads / 32) * (32 / W) * R;
    const uint64_t need = (m + per_cta - 1) / per_cta;
    uint64_t g = 0;
    cudaError_t e = plan_grid((const void*)kern, threads, smem, grid, need, carveout_for(smem, threads), &g, uns);
    if (e != cudaSuccess || *uns) return e;
    kern<<<(unsigned)g, threads, smem, s>>>(*(const KaryParams<K>*)params, (const K*)q, m, (O*)out);
    count_launch();
    return cudaGetLastError();
}

template <class K, class O>
static cudaError_t dispatch_kary(const void* params, const void* q, uint64_t m, void* out, uint32_t threads,
                                 uint32_t W, uint32_t R, Grid grid, uint32_t smem, cudaStream_t s,
                                 bool* uns) {
#define BS_KARY_R(WW)                                                                         \
    case WW:                                                                                  \
        switch (R) {                                                                          \
            case 1: return go_kary<K, O, WW, 1>(params, q, m, out, threads, grid, smem, s, uns); \
            case 2: return go_kary<K, O, WW, 2>(params, q, m, out, threads, grid, smem, s, uns); \
            case 4: return go_kary<K, O, WW, 4>(params, q, m, out, threads, grid, smem, s, uns); \
            case 8: return go_kary<K, O, WW, 8>(params, q, m, out, threads, grid, smem, s, uns); \
            default: *uns = true; return cudaSuccess;                                         \
        }
    switch (W) {
        BS_KARY_R(2)
        BS_KARY_R(4)
        BS_KARY_R(8)
        BS_KARY_R(16)
        BS_KARY_R(32)
        default: *uns = true; return cudaSuccess;
    }
#undef BS_KARY_R
}

cudaError_t launch_kary(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                        uint32_t threads, uint32_t W, uint32_t R, Grid grid, uint32_t smem,
                        cudaStream_t s, bool* uns) {
    *uns = false;
    if (kb == 8 && ob == 8) return dispatch_kary<uint64_t, uint64_t>(params, q, m, out, threads, W, R, grid, smem, s, uns);
    if (kb == 8 && ob == 4) return dispatch_kary<uint64_t, uint32_t>(params, q, m, out, threads, W, R, grid, smem, s, uns);
    if (kb == 4 && ob == 8) return dispatch_kary<uint32_t, uint64_t>(params, q, m, out, threads, W, R, grid, smem, s, uns);
    return dispatch_kary<uint32_t, uint32_t>(params, q, m, out, threads, W, R, grid, smem, s, uns);
}

}  // namespace bs
