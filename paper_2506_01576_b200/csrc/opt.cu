// opt.cu — "BS (all optimizations)", §4.4 Listing 2,
// re-designed for sm_100a (DESIGN.md §"OPT kernel"):
//
//   §4.1 scheduling: persistent grid of SMs x ctas_per_sm CTAs, CTA b
//        owns tiles b, b+grid, ...  (Listing 2 l.6-8, lookup_stride), or one
//        tile per CTA on the hardware scheduler (dynamic).
//   §4.2 pinning: the first D levels of the offset search (+ a
//        prefix of level D, "full-pinning") are staged ONCE per CTA into shared
//        memory by TMA bulk copies (Listing 2 l.3 extract_into_scratch), from a
//        level-major table built by bs_build:  T[base_d + k] = a[n-1-(2k+1)s_d].
//        Level-major instead of the paper's ascending order: same entries
//        (P:119's positions), but a probe at level d is T[base_d + k] with k the
//        bits taken so far, so the top levels are broadcasts and deeper levels
//        spread over banks instead of power-of-two strides (SURVEY TL;DR 4).
//   §4.3 reordering: a tile of NT*NREG lookups is bucketed in
//        shared memory by its leading key bits (one counting/radix pass,
//        digit = (q - kmin) >> shift), each thread then takes sorted elements
//        r*NT + tid; results are either written straight to their original
//        slot (lookup-reordering) or scattered back through shared memory and
//        stored coalesced (full-reordering, Listing 2 l.35-39).
//   Global phase (Listing 1 loop, reading R11: on the sorted array): each
//        thread advances its NREG lookups one level at a time, so NREG
//        independent loads are in flight per thread.
#include "common.cuh"
#include "params.h"

namespace bs {

constexpr uint32_t kMiscBytes = 256;   // mbarrier (16 B) + 32 warp sums

template <class K>
__device__ __forceinline__ uint32_t bucket_of(K key, K kmin, uint32_t shift, uint32_t nb) {
    if (key <= kmin) return 0;
    const uint64_t d = (uint64_t)((K)(key - kmin) >> shift);
    return d < nb ? (uint32_t)d : nb - 1;
}

// Exclusive scan of hist[0 .. NT*NREG) in place; thread t owns entries
// [t*NREG, (t+1)*NREG).  wsum: >= 32 u32 of shared scratch.
template <int NREG>
__device__ __forceinline__ void block_exclusive_scan(uint32_t* hist, uint32_t* wsum) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    uint32_t loc[NREG];
    uint32_t sum = 0;
#pragma unroll
    for (int r = 0; r < NREG; ++r) { loc[r] = hist[tid * NREG + r]; sum += loc[r]; }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nwarps ? wsum[lane] : 0;
        uint32_t s = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= (uint32_t)o) s += y;
        }
        if (lane < nwarps) wsum[lane] = s - w;   // exclusive warp offsets
    }
    __syncthreads();
    uint32_t run = wsum[warp] + x - sum;
#pragma unroll
    for (int r = 0; r < NREG; ++r) { hist[tid * NREG + r] = run; run += loc[r]; }
}

template <class K, class O, int NREG, int REORDER>
__global__ void k_bs_opt(const OptParams<K> p, const K* __restrict__ q, uint64_t m, O* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t NT = blockDim.x, tid = threadIdx.x;
    const uint32_t tile = NT * NREG;
    K* T = reinterpret_cast<K*>(smem);                                  // pinned table
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.tab_bytes);
    uint32_t* wsum = reinterpret_cast<uint32_t*>(smem + p.tab_bytes + 16);
    unsigned char* buf = smem + p.tab_bytes + kMiscBytes;
    K* skeys = reinterpret_cast<K*>(buf);                               // tile keys
    O* sres = reinterpret_cast<O*>(buf + (size_t)tile * sizeof(K));     // tile results
    uint32_t* hist = reinterpret_cast<uint32_t*>(buf + (size_t)tile * (sizeof(K) + sizeof(O)));
    uint16_t* sslot = reinterpret_cast<uint16_t*>(hist + tile);         // sort permutation

    // Listing 2 l.3: extract_into_scratch — one TMA bulk copy per CTA.
    if (p.tab_bytes) stage_to_smem(T, p.tab, p.tab_bytes, bar);

    const uint64_t pol = policy_evict_first();
    const bool sh = p.stream_hint != 0;
    const uint64_t n = p.n;
    const uint64_t sD = (p.D < p.levels) ? (p.s0 >> p.D) : 0;     // first global step
    const uint64_t sDm1 = (p.D > 0) ? (p.s0 >> (p.D - 1)) : 0;
    const uint64_t ntiles = (m + tile - 1) / tile;

    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {  // l.8 while lookup_offset < len
        const uint64_t base = t * tile;
        K key[NREG];
        uint32_t slot[NREG];
        // l.10-11: pre-fetch NREG lookups per thread, coalesced per register
#pragma unroll
        for (int r = 0; r < NREG; ++r) {
            const uint64_t i = base + (uint64_t)r * NT + tid;
            key[r] = (i < m) ? load_stream(q + i, sh, pol) : KeyMax<K>::v;
            slot[r] = r * NT + tid;
        }
        if (REORDER) {
            // l.13 block_sort(l): one counting pass over `tile` buckets.
            for (uint32_t b = tid; b < tile; b += NT) hist[b] = 0;
            __syncthreads();
            uint32_t dig[NREG], rank[NREG];
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                dig[r] = bucket_of<K>(key[r], p.kmin, p.shift, tile);
                rank[r] = atomicAdd(&hist[dig[r]], 1u);
            }
            __syncthreads();
            block_exclusive_scan<NREG>(hist, wsum);
            __syncthreads();
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                const uint32_t dst = hist[dig[r]] + rank[r];
                skeys[dst] = key[r];
                sslot[dst] = (uint16_t)slot[r];
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                key[r] = skeys[r * NT + tid];
                slot[r] = sslot[r * NT + tid];
            }
        }

        // ---- pinned phase (l.17-27) on the level-major table ----
        uint32_t kk[NREG];
        K v[NREG];
#pragma unroll
        for (int r = 0; r < NREG; ++r) { kk[r] = 0; v[r] = p.a_last; }
        for (uint32_t d = 0; d < p.D; ++d) {
            const uint32_t vd = p.valid[d];
            const K* Td = T + p.base[d];
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                const uint32_t k = kk[r];
                const K x = Td[k < vd ? k : vd - 1];
                const bool b = (k < vd) && (x >= key[r]);   // guard "step <= offset" + probe
                kk[r] = 2 * k + (b ? 1u : 0u);
                v[r] = b ? x : v[r];
            }
        }
        // l.29-31: map to the global offset; next step s_D
        uint64_t off[NREG];
        uint32_t skip = 0;   // bit r: level D already resolved from the partial prefix
#pragma unroll
        for (int r = 0; r < NREG; ++r) off[r] = n - 1 - (uint64_t)kk[r] * sDm1;
        if (p.P) {   // l.23-27 (reading R10): partial level D ("full-pinning")
            const K* TD = T + p.base[p.D];
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                const uint32_t k = kk[r];
                const bool in = k < p.P;
                const K x = TD[in ? k : p.P - 1];
                if (in) {
                    skip |= 1u << r;
                    if (x >= key[r]) { off[r] -= sD; v[r] = x; }
                }
            }
        }
        // ---- global phase (l.33, reading R11): Listing 1 loop, NREG loads in flight ----
        // upper global levels (step >= l1_step) with L1-allocating loads, as the
        // naive kernel gets them; the deep levels with L1::no_allocate (+ hints)
        auto global_step = [&](uint64_t step, bool l1) {
            const bool hint = p.leaf_hint && step < p.evict_step;
            const bool first = (step == sD);
            K x[NREG];
            bool go[NREG];
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                go[r] = (step <= off[r]) && !(first && ((skip >> r) & 1u));
                if (l1) x[r] = go[r] ? ldg(p.a + (off[r] - step)) : (K)0;
                else x[r] = go[r] ? load_key(p.a + (off[r] - step), hint, pol) : (K)0;
            }
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                if (go[r] && x[r] >= key[r]) { off[r] -= step; v[r] = x[r]; }
            }
        };
        uint64_t step = sD;
        for (; step > 0 && step >= p.l1_step; step >>= 1) global_step(step, true);
        for (; step > 0; step >>= 1) global_step(step, false);

        // ---- results (l.35-39) ----
        if (REORDER == 2) {
#pragma unroll
            for (int r = 0; r < NREG; ++r) sres[slot[r]] = encode<O>(off[r], v[r], key[r], n);
            __syncthreads();
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                const uint64_t i = base + (uint64_t)r * NT + tid;
                if (i < m) store_stream(out + i, sres[r * NT + tid], sh, pol);
            }
        } else {
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                const uint64_t i = base + slot[r];
                if (i < m) store_stream(out + i, encode<O>(off[r], v[r], key[r], n), sh, pol);
            }
        }
    }
}

uint32_t opt_smem_extra(int kb, int ob, uint32_t threads, uint32_t nreg, uint32_t reorder) {
    const uint32_t tile = threads * nreg;
    uint32_t b = kMiscBytes;
    if (reorder) b += tile * (uint32_t)(kb + ob + 4 + 2);
    return (b + 15u) & ~15u;
}

template <class K, class O, int NREG, int RE>
static cudaError_t go_opt(const void* params, const void* q, uint64_t m, void* out, uint32_t threads,
                          Grid grid, uint32_t smem, cudaStream_t s, bool* unsupported) {
    auto kern = k_bs_opt<K, O, NREG, RE>;
    const uint64_t tile = (uint64_t)threads * NREG;
    const uint64_t ntiles = (m + tile - 1) / tile;
    uint64_t g = 0;
    cudaError_t e = plan_grid((const void*)kern, threads, smem, grid, ntiles, carveout_for(smem, threads), &g, unsupported);
    if (e != cudaSuccess || *unsupported) return e;
    kern<<<(unsigned)g, threads, smem, s>>>(*(const OptParams<K>*)params, (const K*)q, m, (O*)out);
    count_launch();
    return cudaGetLastError();
}

template <class K, class O>
static cudaError_t dispatch_opt(const void* params, const void* q, uint64_t m, void* out, uint32_t threads,
                                uint32_t nreg, uint32_t reorder, Grid grid, uint32_t smem,
                                cudaStream_t s, bool* uns) {
#define BS_OPT_CASE(NR)                                                                          \
    case NR:                                                                                     \
        if (reorder == 0) return go_opt<K, O, NR, 0>(params, q, m, out, threads, grid, smem, s, uns); \
        if (reorder == 1) return go_opt<K, O, NR, 1>(params, q, m, out, threads, grid, smem, s, uns); \
        return go_opt<K, O, NR, 2>(params, q, m, out, threads, grid, smem, s, uns);
    switch (nreg) {
        BS_OPT_CASE(1)
        BS_OPT_CASE(2)
        BS_OPT_CASE(4)
        BS_OPT_CASE(8)
        BS_OPT_CASE(16)
        default: *uns = true; return cudaSuccess;
    }
#undef BS_OPT_CASE
}

cudaError_t launch_opt(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                       uint32_t threads, uint32_t nreg, uint32_t reorder, Grid grid,
                       uint32_t smem, cudaStream_t s, bool* uns) {
    *uns = false;
    if (kb == 8 && ob == 8) return dispatch_opt<uint64_t, uint64_t>(params, q, m, out, threads, nreg, reorder, grid, smem, s, uns);
    if (kb == 8 && ob == 4) return dispatch_opt<uint64_t, uint32_t>(params, q, m, out, threads, nreg, reorder, grid, smem, s, uns);
    if (kb == 4 && ob == 8) return dispatch_opt<uint32_t, uint64_t>(params, q, m, out, threads, nreg, reorder, grid, smem, s, uns);
    return dispatch_opt<uint32_t, uint32_t>(params, q, m, out, threads, nreg, reorder, grid, smem, s, uns);
}

}  // namespace bs
