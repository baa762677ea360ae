// seg.cu — segment-staged lookup for ordered query batches (BS_REORDER_SORTED).
//
// PAPER.md §4.3 / Fig. 1b: when the lookups arrive sorted,
// neighbouring lookups share their search paths, and binary search becomes the
// fastest index of all.  The K-ary kernel cannot cash that in on B200: its
// issue cost per lookup is the same in any order.  This
// kernel turns the ordering into locality explicitly:
//
//  * the sorted array is cut into segments of S = 2^D keys; segment b holds
//    positions [b*S, b*S + S), and its queries are those with
//    a[b*S - 1] < q <= a[b*S + S - 1] (the first and last segment are open);
//  * CTA c owns the segments [B*c/G, B*(c+1)/G); its threads first find the
//    query range of each of them by bisection over the query batch
//    (#queries <= a[b*S - 1]; monotone in the key for ANY batch order, so the
//    ranges always tile [0, m));
//  * per segment the CTA stages ONE 32-bit order-preserving image of the keys
//    into shared memory, in Eytzinger (BFS) order — F(x) = (x - seg_min) >> sh,
//    sh chosen per segment so the segment's span fits 31 bits (exact, sh = 0,
//    whenever the span is < 2^31: every u32 segment, and u64 segments of
//    narrow key ranges — so keys sharing their high word cost nothing);
//  * each query descends D levels of the image (one 4-B shared load per level,
//    level d's probes on the contiguous slots [2^d, 2^(d+1)): no power-of-two
//    bank aliasing), which gives c = #(keys with F < F(q)) <= lb; when sh > 0
//    the exact first key >= q is found from c with one global read of the
//    (L2-hot) segment (galloping over equal images: O(log) reads worst case);
//  * queries outside their range (a batch that is not sorted) take a plain
//    global bisection, so the result contract holds for any order; only the
//    speed needs the order.
//
// One global read per query (its key), one write (its result), and each
// segment read once per batch: the pre-sorted roofline of SURVEY.md §8d
// (key + out + n*key/m bytes per lookup).
#include "common.cuh"
#include "params.h"

namespace bs {

// #(i : q[i] <= x) by bisection over an arbitrary batch (monotone in x)
template <class K>
__device__ __forceinline__ uint64_t upper_bound_any(const K* __restrict__ q, uint64_t m, K x) {
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (ldg(q + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// #(i : a[i] < x): the plain lower bound, for queries outside their segment
template <class K>
__device__ __forceinline__ uint64_t lower_bound_global(const K* __restrict__ a, uint64_t n, K x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (ldg(a + mid) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// order-preserving 32-bit image of x relative to a segment: 0 below its minimum
template <class K>
__device__ __forceinline__ uint32_t seg_image(K x, K smin, uint32_t sh) {
    if (x <= smin) return 0u;
    const uint64_t d = (uint64_t)(x - smin) >> sh;
    return d > 0x80000000ull ? 0x80000000u : (uint32_t)d;
}

template <class K, int D, int OB>
__global__ void __launch_bounds__(1024, 1)
k_seg_sorted(const SegParams<K> p) {
    constexpr uint32_t S = 1u << D;
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* F = sm;                                         // slot 0: segment max; 1..S-1: Eytzinger
    uint64_t* bnd = reinterpret_cast<uint64_t*>(sm + S);      // query ranges of this CTA's segments
    const uint64_t G = gridDim.x, B = p.B, n = p.n, m = p.m;
    const uint64_t b0 = B * blockIdx.x / G, b1 = B * (blockIdx.x + 1) / G;
    const uint32_t nb = (uint32_t)(b1 - b0);
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    constexpr uint64_t MISS = 1ull << (8 * OB - 1);

    for (uint32_t i = threadIdx.x; i <= nb; i += blockDim.x) {
        const uint64_t b = b0 + i;
        bnd[i] = b == 0 ? 0 : b >= B ? m : upper_bound_any(p.q, m, ldg(p.a + b * S - 1));
    }
    for (uint64_t b = b0; b < b1; ++b) {
        const uint64_t lo = b * S;
        const uint32_t len = (uint32_t)((n - lo) < S ? (n - lo) : S);
        const K* seg = p.a + lo;
        const K smin = ldg(seg), smax = ldg(seg + len - 1);
        const uint64_t span = (uint64_t)(smax - smin);
        const uint32_t bl = span ? 64u - (uint32_t)__clzll((long long)span) : 0u;
        const uint32_t sh = bl > 31u ? bl - 31u : 0u;
        __syncthreads();   // previous segment's searches are done with F (and bnd is written)
        for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
            // past the segment end: above every in-range query's image (<= 2^31)
            const uint32_t f = i < len ? seg_image(ldg(seg + i), smin, sh) : 0xFFFFFFFFu;
            uint32_t slot = 0;
            if (i != S - 1) {
                const uint32_t j = i + 1, t = (uint32_t)__ffs((int)j) - 1u;
                slot = (1u << (D - 1 - t)) + (j >> (t + 1));
            }
            F[slot] = f;
        }
        __syncthreads();
        const K lower = b ? ldg(p.a + lo - 1) : (K)0;
        const bool first = b == 0, last = b == B - 1;
        const uint64_t q0 = bnd[b - b0], q1 = bnd[b - b0 + 1];
        for (uint64_t i = q0 + threadIdx.x; i < q1; i += blockDim.x) {
            const K x = load_stream(p.q + i, true, pol_stream);
            uint64_t lb;
            bool hit;
            if ((first || x > lower) && (last || x <= smax)) {
                const uint32_t fx = seg_image(x, smin, sh);
                uint32_t k = 1;
#pragma unroll
                for (int d = 0; d < D; ++d) k = 2u * k + (F[k] < fx ? 1u : 0u);
                uint32_t c = k - S;                  // keys whose image is below q's: <= lb - lo
                K v;
                if (sh == 0) {
                    // exact image: the successor is the last left turn (slot 0 = segment max)
                    v = c < len ? (K)(smin + (K)F[k >> __ffs((int)~k)]) : (K)0;
                    // only the segment max (slot 0, not in the tree) can be below q here:
                    // the last segment's queries above every key
                    if (c < len && v < x) c = len;
                } else {
                    v = c < len ? ldg(seg + c) : (K)0;
                    if (c < len && v < x) {
                        // keys sharing q's image: gallop, then bisect (seg[c] < x)
                        uint32_t l = c + 1, step = 1, h;
                        for (;;) {
                            h = l - 1 + step;
                            if (h >= len) { h = len; break; }
                            if (ldg(seg + h) >= x) break;
                            l = h + 1;
                            step <<= 1;
                        }
                        while (l < h) {
                            const uint32_t mid = (l + h) >> 1;
                            if (ldg(seg + mid) < x) l = mid + 1;
                            else h = mid;
                        }
                        c = l;
                        v = c < len ? ldg(seg + c) : (K)0;
                    }
                }
                lb = lo + c;
                hit = c < len && v == x;
            } else {
                lb = lower_bound_global(p.a, n, x);
                hit = lb < n && ldg(p.a + lb) == x;
            }
            const uint64_t r = hit ? lb : (lb | MISS);
            if constexpr (OB == 8) store_stream((uint64_t*)p.out + i, r, true, pol_stream);
            else store_stream((uint32_t*)p.out + i, (uint32_t)r, true, pol_stream);
        }
    }
}

constexpr int kSegLog2 = 13;   // S = 8192 keys per segment: a 32-KB image

static uint64_t seg_smem_bytes(uint64_t n, uint32_t grid) {
    const uint64_t S = 1ull << kSegLog2;
    const uint64_t B = (n + S - 1) / S;
    const uint64_t nb = (B + grid - 1) / grid + 1;
    return S * 4 + nb * 8 + 16;
}

template <class K, int D, int OB>
static cudaError_t go_seg(const SegParams<K>& p, Grid grid, cudaStream_t s, bool* uns) {
    auto kern = k_seg_sorted<K, D, OB>;
    const uint32_t threads = 1024;
    uint64_t g = 0;
    grid.sched_static = 1;
    grid.ctas_per_sm = 1;
    const uint32_t smem = (uint32_t)seg_smem_bytes(p.n, grid.sm_count);
    cudaError_t e = plan_grid((const void*)kern, threads, smem, grid, grid.sm_count, carveout_for(smem, threads), &g, uns);
    if (e != cudaSuccess || *uns) return e;
    kern<<<(unsigned)g, threads, smem, s>>>(p);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_seg_sorted(int kb, int ob, const void* a, uint64_t n, const void* q, uint64_t m, void* out,
                              uint32_t stream_hint, Grid grid, cudaStream_t s, bool* uns) {
    constexpr int D = kSegLog2;
    const uint64_t S = 1ull << D;
    if (seg_smem_bytes(n, grid.sm_count) > 200u * 1024u) { *uns = true; return cudaSuccess; }
    if (kb == 8) {
        SegParams<uint64_t> p{(const uint64_t*)a, n, (const uint64_t*)q, m, out, (uint32_t)ob, (n + S - 1) / S, stream_hint};
        return ob == 8 ? go_seg<uint64_t, D, 8>(p, grid, s, uns) : go_seg<uint64_t, D, 4>(p, grid, s, uns);
    }
    SegParams<uint32_t> p{(const uint32_t*)a, n, (const uint32_t*)q, m, out, (uint32_t)ob, (n + S - 1) / S, stream_hint};
    return ob == 8 ? go_seg<uint32_t, D, 8>(p, grid, s, uns) : go_seg<uint32_t, D, 4>(p, grid, s, uns);
}

}  // namespace bs
