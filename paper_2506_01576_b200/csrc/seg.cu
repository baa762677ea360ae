// seg.cu — segment-staged lookups: ordered batches (BS_REORDER_SORTED) and the
// global partition of a random batch (BS_REORDER_GLOBAL).
//
// PAPER.md §4.3 / Fig. 1b: when the lookups arrive sorted,
// neighbouring lookups share their search paths, and binary search becomes the
// fastest index of all; sorting the batch globally is the paper's reference
// point for its cheap local reordering ("out-of-place", "too expensive",
// P:133-135).  On B200 the K-ary kernel cannot cash in on an ordered batch —
// its issue cost per lookup is the same in any order — and a
// random batch is bound by one random 128-B DRAM line per lookup (the DRAM atom,
// profiles/r2a_ubench_gather2.json).  These kernels turn order into locality:
//
//  * the sorted array is cut into segments of S = 2^D keys; segment b holds
//    positions [b*S, b*S + S), and its queries are those with
//    a[b*S - 1] < q <= a[b*S + S - 1] (the first and last segment are open);
//  * per segment a CTA stages ONE 32-bit order-preserving image of the keys
//    into shared memory, in Eytzinger (BFS) order — F(x) = (x - seg_min) >> sh,
//    sh chosen per segment so the segment's span fits 31 bits (exact, sh = 0,
//    whenever the span is < 2^31: every u32 segment, and u64 segments of
//    narrow key ranges — keys sharing their high word cost nothing);
//  * each query descends D levels of the image (one 4-B shared load per level,
//    level d's probes on the contiguous slots [2^d, 2^(d+1)): no power-of-two
//    bank aliasing), which gives c = #(keys with F < F(q)) <= lb; when sh > 0
//    the exact first key >= q is found from c with one global read of the
//    (L2-hot) segment (galloping over equal images: O(log) reads worst case).
//
// SORTED: CTA c owns segments [B*c/G, B*(c+1)/G) and finds each one's query
// range by bisection over the batch (#queries <= a[b*S - 1]: monotone in the key
// for ANY batch order, so the ranges tile [0, m)); a query outside its range (an
// unsorted batch) takes a plain global bisection — correct in any order, fast
// only when ordered.
//
// GLOBAL (a random batch; caller's workspace):
//   k_part     per tile of T = 8192 queries: bucket b(q) = #(segment maxima < q)
//              (a shared-memory Eytzinger image of the maxima + an exact check);
//              a counting sort of the tile by bucket in shared memory gives each
//              query its slot `dst` in the tile's bucket-grouped order (the slot
//              permutation goes to `slot2`); one global atomic per query reserves
//              its place in bucket b's region of the record array (q, dst);
//              regions hold cap = 1.25 m/B + 64 records, the rest overflows to a
//              list (a skewed batch stays correct, only slower);
//   k_seg_part the segment lookup per bucket over its records; the result goes
//              to res2[dst] (the tile's bucket-grouped order: the CTAs working on
//              neighbouring buckets fill each tile's window together in L2);
//   k_part_ovf overflowed records, by global bisection;
//   k_unpart   per tile: res2 and slot2 in, results scattered back to query
//              order in shared memory, one coalesced store (Listing 2 l.35-39's
//              "unsort", at batch scale).
#include <cstring>
#include <type_traits>

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

// order-preserving 32-bit image of x relative to `base`: 0 at or below it
template <class K>
__device__ __forceinline__ uint32_t seg_image(K x, K base, uint32_t sh) {
    if (x <= base) return 0u;
    const uint64_t d = (uint64_t)(x - base) >> sh;
    return d > 0x80000000ull ? 0x80000000u : (uint32_t)d;
}

// shift that makes the image of [lo, hi] fit 31 bits
template <class K>
__device__ __forceinline__ uint32_t image_shift(K lo, K hi) {
    const uint64_t span = (uint64_t)(hi - lo);
    const uint32_t bl = span ? 64u - (uint32_t)__clzll((long long)span) : 0u;
    return bl > 31u ? bl - 31u : 0u;
}

// Eytzinger slot of sorted position i (< 2^D - 1) in a tree of 2^D - 1 nodes
template <int D>
__device__ __forceinline__ uint32_t eytz_slot(uint32_t i) {
    const uint32_t j = i + 1, t = (uint32_t)__ffs((int)j) - 1u;
    return (1u << (D - 1 - t)) + (j >> (t + 1));
}

// Stage segment [seg, seg + len) as its image: slot 0 = element S-1 (the
// segment max, outside the tree), slots 1..S-1 = elements 0..S-2; past len:
// 0xFFFFFFFF (above every in-range query).  Caller synchronises.
template <class K, int D>
__device__ __forceinline__ void stage_segment(uint32_t* F, const K* __restrict__ seg, uint32_t len, K smin, uint32_t sh) {
    constexpr uint32_t S = 1u << D;
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
        const uint32_t f = i < len ? seg_image(ldg(seg + i), smin, sh) : 0xFFFFFFFFu;
        F[i == S - 1 ? 0u : eytz_slot<D>(i)] = f;
    }
}

// lb - (segment start) and the hit flag of an in-range query x
template <class K, int D>
__device__ __forceinline__ uint32_t seg_search(const uint32_t* F, const K* __restrict__ seg, uint32_t len, K smin,
                                               uint32_t sh, K x, bool* hit) {
    constexpr uint32_t S = 1u << D;
    const uint32_t fx = seg_image(x, smin, sh);
    uint32_t k = 1;
#pragma unroll
    for (int d = 0; d < D; ++d) k = 2u * k + (F[k] < fx ? 1u : 0u);
    uint32_t c = k - S;                  // keys whose image is below q's: <= lb - seg start
    K v;
    if (sh == 0) {
        // exact image: the successor is the last left turn (slot 0 = segment max)
        v = c < len ? (K)(smin + (K)F[k >> __ffs((int)~k)]) : (K)0;
        // only the segment max (slot 0, outside the tree) can be below q here:
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
    *hit = c < len && v == x;
    return c;
}

template <int OB>
__device__ __forceinline__ uint64_t enc(uint64_t lb, bool hit) {
    constexpr uint64_t MISS = 1ull << (8 * OB - 1);
    return hit ? lb : (lb | MISS);
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

    for (uint32_t i = threadIdx.x; i <= nb; i += blockDim.x) {
        const uint64_t b = b0 + i;
        bnd[i] = b == 0 ? 0 : b >= B ? m : upper_bound_any(p.q, m, ldg(p.a + b * S - 1));
    }
    for (uint64_t b = b0; b < b1; ++b) {
        const uint64_t lo = b * S;
        const uint32_t len = (uint32_t)((n - lo) < S ? (n - lo) : S);
        const K* seg = p.a + lo;
        const K smin = ldg(seg), smax = ldg(seg + len - 1);
        const uint32_t sh = image_shift(smin, smax);
        __syncthreads();   // previous segment's searches are done with F (and bnd is written)
        stage_segment<K, D>(F, seg, len, smin, sh);
        __syncthreads();
        const K lower = b ? ldg(p.a + lo - 1) : (K)0;
        const bool first = b == 0, last = b == B - 1;
        const uint64_t q0 = bnd[b - b0], q1 = bnd[b - b0 + 1];
        for (uint64_t i = q0 + threadIdx.x; i < q1; i += blockDim.x) {
            const K x = load_stream(p.q + i, true, pol_stream);
            uint64_t lb;
            bool hit;
            if ((first || x > lower) && (last || x <= smax)) {
                lb = lo + seg_search<K, D>(F, seg, len, smin, sh, x, &hit);
            } else {
                lb = lower_bound_global(p.a, n, x);
                hit = lb < n && ldg(p.a + lb) == x;
            }
            const uint64_t r = enc<OB>(lb, hit);
            if constexpr (OB == 8) store_stream((uint64_t*)p.out + i, r, true, pol_stream);
            else store_stream((uint32_t*)p.out + i, (uint32_t)r, true, pol_stream);
        }
    }
}

// ---------------------------------------------------------------- GLOBAL mode

constexpr int kSegLog2 = 13;           // S = 8192 keys per segment: a 32-KB image
constexpr uint32_t kPartTile = 8192;   // queries per partition tile (slot2 is u16)
constexpr uint32_t kPartLog2SB = 13;   // at most 2^13 bucket groups in a tile's counting sort
constexpr uint32_t kPartMaxLog2B = 14; // buckets <= 2^14: the maxima image fits shared memory (64 KB)

template <class K> struct PartRec;
template <> struct __align__(16) PartRec<uint64_t> { uint64_t q; uint32_t dst; uint32_t pad; };
template <> struct PartRec<uint32_t> { uint32_t q; uint32_t dst; };

template <class K>
struct PartParams {
    const K* a;
    uint64_t n, m;
    const K* q;
    void* out;
    uint64_t B;               // segments
    uint32_t DB;              // log2 of the maxima tree size (2^DB >= B)
    uint32_t sbsh;            // bucket -> bucket group shift (tile counting sort)
    uint64_t cap;             // records per bucket region
    uint32_t* cursor;         // [B] reservations
    uint32_t* ovf_n;          // overflowed records
    PartRec<K>* rec;          // [B * cap]
    PartRec<K>* ovf;          // [m]
    void* res2;               // [m] results in each tile's bucket-grouped order
    uint16_t* slot2;          // [m] tile slot of each res2 entry
    uint32_t stream_hint;
};

// bucket of x: #(segment maxima < x), maxima max_c = a[(c+1)*S - 1], c < B-1
template <class K, int D>
__device__ __forceinline__ uint32_t part_bucket(const uint32_t* MF, uint32_t DB, const K* __restrict__ a, uint64_t B,
                                                K gbase, uint32_t gsh, K x) {
    constexpr uint64_t S = 1ull << D;
    const uint32_t fx = seg_image(x, gbase, gsh);
    uint32_t k = 1;
    for (uint32_t d = 0; d < DB; ++d) k = 2u * k + (MF[k] < fx ? 1u : 0u);
    uint32_t c = k - (1u << DB);              // maxima whose image is below q's: <= bucket
    const uint32_t nm = (uint32_t)(B - 1);   // maxima in the table
    if (c < nm && ldg(a + ((uint64_t)c + 1) * S - 1) < x) {
        uint32_t l = c + 1, step = 1, h;
        for (;;) {
            h = l - 1 + step;
            if (h >= nm) { h = nm; break; }
            if (ldg(a + ((uint64_t)h + 1) * S - 1) >= x) break;
            l = h + 1;
            step <<= 1;
        }
        while (l < h) {
            const uint32_t mid = (l + h) >> 1;
            if (ldg(a + ((uint64_t)mid + 1) * S - 1) < x) l = mid + 1;
            else h = mid;
        }
        c = l;
    }
    return c;
}

// block-wide exclusive scan of cnt[0..N) in place (blockDim.x = 1024)
__device__ __forceinline__ void block_exscan(uint32_t* cnt, uint32_t N, uint32_t* warp_tmp) {
    const uint32_t per = (N + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per;
    uint32_t s = 0;
    for (uint32_t i = 0; i < per; ++i)
        if (b0 + i < N) s += cnt[b0 + i];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
    }
    if (lane == 31) warp_tmp[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t v = lane < (blockDim.x >> 5) ? warp_tmp[lane] : 0u;
        uint32_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= (uint32_t)o) wi += y;
        }
        warp_tmp[lane] = wi - v;
    }
    __syncthreads();
    uint32_t run = warp_tmp[w] + inc - s;
    for (uint32_t i = 0; i < per; ++i) {
        if (b0 + i < N) {
            const uint32_t c = cnt[b0 + i];
            cnt[b0 + i] = run;
            run += c;
        }
    }
    __syncthreads();
}

template <class K, int D>
__global__ void __launch_bounds__(1024, 1)
k_part(const PartParams<K> p) {
    constexpr uint32_t E = kPartTile / 1024;   // queries per thread per tile
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t DB = p.DB, NT = 1u << DB;
    const uint32_t NSB = (uint32_t)((p.B - 1) >> p.sbsh) + 1;
    const bool exact_groups = p.sbsh == 0;      // bucket groups are buckets: one reservation per (tile, bucket)
    uint32_t* MF = sm;                          // [NT] maxima image (Eytzinger, slot 0 unused)
    uint32_t* cnt = MF + NT;                    // [NSB] counts, then running ranks
    uint32_t* off = cnt + NSB;                  // [NSB] tile offsets of the groups
    uint32_t* gb = off + NSB;                   // [NSB] reserved base in the bucket region (exact groups)
    uint32_t* warp_tmp = gb + NSB;              // [32]
    constexpr uint64_t S = 1ull << D;
    const K gbase = ldg(p.a), gtop = ldg(p.a + p.n - 1);
    const uint32_t gsh = image_shift(gbase, gtop);
    for (uint32_t k = threadIdx.x; k < NT; k += blockDim.x) {
        uint32_t f = 0xFFFFFFFFu;
        if (k > 0) {
            // slot k at depth d holds sorted maximum i = (2(k - 2^d) + 1) 2^(DB-1-d) - 1
            const uint32_t d = 31u - (uint32_t)__clz((int)k);
            const uint64_t i = ((2ull * (k - (1u << d)) + 1) << (DB - 1 - d)) - 1;
            if (i < p.B - 1) f = seg_image(ldg(p.a + (i + 1) * S - 1), gbase, gsh);
        }
        MF[k] = f;
    }
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t ntiles = (p.m + kPartTile - 1) / kPartTile;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (uint32_t i = threadIdx.x; i < NSB; i += blockDim.x) cnt[i] = 0;
        __syncthreads();   // (also: the maxima image is complete)
        K x[E];
        uint32_t b[E];
        const uint64_t base = t * kPartTile;
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            const uint64_t i = base + e * 1024u + threadIdx.x;
            b[e] = 0xFFFFFFFFu;
            x[e] = 0;
            if (i < p.m) {
                x[e] = load_stream(p.q + i, true, pol_stream);
                b[e] = part_bucket<K, D>(MF, DB, p.a, p.B, gbase, gsh, x[e]);
                atomicAdd(&cnt[b[e] >> p.sbsh], 1u);
            }
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < NSB; i += blockDim.x) off[i] = cnt[i];
        __syncthreads();
        block_exscan(off, NSB, warp_tmp);
        // one global reservation per (tile, bucket): the tile's records of bucket
        // b take [gb[b], gb[b] + cnt[b]) of b's region
        for (uint32_t i = threadIdx.x; i < NSB; i += blockDim.x) {
            const uint32_t c = cnt[i];
            if (exact_groups && c) gb[i] = atomicAdd(p.cursor + i, c);
            cnt[i] = 0;
        }
        __syncthreads();
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            if (b[e] == 0xFFFFFFFFu) continue;
            const uint32_t grp = b[e] >> p.sbsh;
            const uint32_t r = atomicAdd(&cnt[grp], 1u);
            const uint32_t pos = off[grp] + r;
            p.slot2[base + pos] = (uint16_t)(e * 1024u + threadIdx.x);
            PartRec<K> rec;
            memset(&rec, 0, sizeof rec);
            rec.q = x[e];
            rec.dst = (uint32_t)(base + pos);
            const uint32_t g = exact_groups ? gb[grp] + r : atomicAdd(p.cursor + b[e], 1u);
            if (g < p.cap) p.rec[b[e] * p.cap + g] = rec;
            else p.ovf[atomicAdd(p.ovf_n, 1u)] = rec;
        }
        __syncthreads();   // cnt / off / gb are reused by the next tile
    }
}

template <class K, int D, int OB>
__global__ void __launch_bounds__(1024, 1)
k_seg_part(const PartParams<K> p) {
    constexpr uint32_t S = 1u << D;
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* F = sm;
    const uint64_t G = gridDim.x, B = p.B, n = p.n;
    // work items: bucket b split into P parts (P > 1 only when there are fewer
    // buckets than twice the CTAs); CTA c takes items [I*c/G, I*(c+1)/G), so
    // consecutive items of one CTA mostly share their segment
    const uint64_t P = B >= 2 * G ? 1 : (2 * G + B - 1) / B;
    const uint64_t I = B * P;
    const uint64_t i0 = I * blockIdx.x / G, i1 = I * (blockIdx.x + 1) / G;
    uint64_t staged = ~0ull;
    for (uint64_t it = i0; it < i1; ++it) {
        const uint64_t b = it / P, part = it % P;
        const uint64_t lo = b * S;
        const uint32_t len = (uint32_t)((n - lo) < S ? (n - lo) : S);
        const K* seg = p.a + lo;
        const K smin = ldg(seg), smax = ldg(seg + len - 1);
        const uint32_t sh = image_shift(smin, smax);
        if (b != staged) {
            __syncthreads();
            stage_segment<K, D>(F, seg, len, smin, sh);
            __syncthreads();
            staged = b;
        }
        uint32_t cntb = p.cursor[b];
        if (cntb > p.cap) cntb = (uint32_t)p.cap;
        const uint32_t j0 = (uint32_t)(cntb * part / P), j1 = (uint32_t)(cntb * (part + 1) / P);
        const PartRec<K>* rb = p.rec + b * p.cap;
        for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
            const PartRec<K> r = rb[j];
            bool hit;
            const uint64_t lb = lo + seg_search<K, D>(F, seg, len, smin, sh, r.q, &hit);
            if constexpr (OB == 8) ((uint64_t*)p.res2)[r.dst] = enc<8>(lb, hit);
            else ((uint32_t*)p.res2)[r.dst] = (uint32_t)enc<4>(lb, hit);
        }
    }
}

template <class K, int OB>
__global__ void k_part_ovf(const PartParams<K> p) {
    const uint32_t no = *p.ovf_n;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < no; j += (uint64_t)gridDim.x * blockDim.x) {
        const PartRec<K> r = p.ovf[j];
        const uint64_t lb = lower_bound_global(p.a, p.n, r.q);
        const bool hit = lb < p.n && ldg(p.a + lb) == r.q;
        if constexpr (OB == 8) ((uint64_t*)p.res2)[r.dst] = enc<8>(lb, hit);
        else ((uint32_t*)p.res2)[r.dst] = (uint32_t)enc<4>(lb, hit);
    }
}

template <class K, int OB>
__global__ void __launch_bounds__(1024, 1)
k_unpart(const PartParams<K> p) {
    using O = typename std::conditional<OB == 8, uint64_t, uint32_t>::type;
    extern __shared__ __align__(16) uint32_t sm[];
    O* tile = reinterpret_cast<O*>(sm);
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t ntiles = (p.m + kPartTile - 1) / kPartTile;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t base = t * kPartTile;
        const uint32_t cnt = (uint32_t)((p.m - base) < kPartTile ? (p.m - base) : kPartTile);
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x)
            tile[p.slot2[base + j]] = ((const O*)p.res2)[base + j];
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x)
            store_stream((O*)p.out + base + j, tile[j], true, pol_stream);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launchers

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

// workspace layout of the GLOBAL mode (all offsets 256-B aligned)
struct PartLayout {
    uint64_t B, cap, o_cursor, o_rec, o_ovf, o_res2, o_slot2, total;
};

static uint64_t al256(uint64_t x) { return (x + 255) & ~255ull; }

static bool part_layout(uint64_t n, uint64_t m, int kb, int ob, PartLayout* L) {
    const uint64_t S = 1ull << kSegLog2;
    L->B = (n + S - 1) / S;
    if (L->B > (1ull << kPartMaxLog2B) || m >= (1ull << 32)) return false;
    L->cap = (m + L->B - 1) / L->B;
    L->cap += L->cap / 4 + 64;
    const uint64_t rs = kb == 8 ? 16 : 8;
    const uint64_t mm = m ? m : 1;
    L->o_cursor = 0;
    L->o_rec = al256(4 * (L->B + 1));
    L->o_ovf = L->o_rec + al256(rs * L->B * L->cap);
    L->o_res2 = L->o_ovf + al256(rs * mm);
    L->o_slot2 = L->o_res2 + al256((uint64_t)ob * mm);
    L->total = L->o_slot2 + al256(2 * mm);
    return true;
}

bool part_workspace_bytes(uint64_t n, uint64_t m, int kb, int ob, uint64_t* bytes) {
    PartLayout L;
    if (!part_layout(n, m, kb, ob, &L)) return false;
    *bytes = L.total;
    return true;
}

template <class K, int OB>
static cudaError_t go_part(PartParams<K> p, const PartLayout& L, char* ws, uint32_t sm_count, cudaStream_t s) {
    constexpr int D = kSegLog2;
    p.cursor = (uint32_t*)(ws + L.o_cursor);
    p.ovf_n = p.cursor + L.B;
    p.rec = (PartRec<K>*)(ws + L.o_rec);
    p.ovf = (PartRec<K>*)(ws + L.o_ovf);
    p.res2 = ws + L.o_res2;
    p.slot2 = (uint16_t*)(ws + L.o_slot2);
    p.B = L.B;
    p.cap = L.cap;
    uint32_t lb = 0;
    while ((1ull << lb) < L.B) ++lb;
    p.DB = lb ? lb : 1;
    p.sbsh = lb > kPartLog2SB ? lb - kPartLog2SB : 0;
    const uint32_t nsb = (uint32_t)((L.B - 1) >> p.sbsh) + 1;
    cudaError_t e = cudaMemsetAsync(p.cursor, 0, 4 * (L.B + 1), s);
    if (e != cudaSuccess) return e;
    Grid grid{1u, 1u, sm_count};
    bool uns = false;
    uint64_t g = 0;
    {   // partition
        auto kern = k_part<K, D>;
        const uint32_t smem = 4u * ((1u << p.DB) + 3u * nsb + 32u);
        e = plan_grid((const void*)kern, 1024, smem, grid, sm_count, carveout_for(smem, 1024), &g, &uns);
        if (e != cudaSuccess) return e;
        if (uns) return cudaErrorInvalidConfiguration;
        kern<<<(unsigned)g, 1024, smem, s>>>(p);
        count_launch();
    }
    {   // segment lookups per bucket
        auto kern = k_seg_part<K, D, OB>;
        const uint32_t smem = 4u << D;
        e = plan_grid((const void*)kern, 1024, smem, grid, sm_count, carveout_for(smem, 1024), &g, &uns);
        if (e != cudaSuccess) return e;
        if (uns) return cudaErrorInvalidConfiguration;
        kern<<<(unsigned)g, 1024, smem, s>>>(p);
        count_launch();
    }
    k_part_ovf<K, OB><<<sm_count, 256, 0, s>>>(p);
    count_launch();
    {   // back to query order
        auto kern = k_unpart<K, OB>;
        const uint32_t smem = kPartTile * OB;
        Grid g2{1u, 0u, sm_count};
        e = plan_grid((const void*)kern, 1024, smem, g2, (p.m + kPartTile - 1) / kPartTile, carveout_for(smem, 1024), &g, &uns);
        if (e != cudaSuccess) return e;
        if (uns) return cudaErrorInvalidConfiguration;
        kern<<<(unsigned)g, 1024, smem, s>>>(p);
        count_launch();
    }
    return cudaGetLastError();
}

cudaError_t launch_part_global(int kb, int ob, const void* a, uint64_t n, const void* q, uint64_t m, void* out,
                               uint32_t stream_hint, void* ws, uint64_t ws_bytes, uint32_t sm_count, cudaStream_t s,
                               bool* uns) {
    PartLayout L;
    if (!part_layout(n, m, kb, ob, &L) || ws_bytes < L.total) { *uns = true; return cudaSuccess; }
    if (kb == 8) {
        PartParams<uint64_t> p{};
        p.a = (const uint64_t*)a; p.n = n; p.m = m; p.q = (const uint64_t*)q; p.out = out; p.stream_hint = stream_hint;
        return ob == 8 ? go_part<uint64_t, 8>(p, L, (char*)ws, sm_count, s) : go_part<uint64_t, 4>(p, L, (char*)ws, sm_count, s);
    }
    PartParams<uint32_t> p{};
    p.a = (const uint32_t*)a; p.n = n; p.m = m; p.q = (const uint32_t*)q; p.out = out; p.stream_hint = stream_hint;
    return ob == 8 ? go_part<uint32_t, 8>(p, L, (char*)ws, sm_count, s) : go_part<uint32_t, 4>(p, L, (char*)ws, sm_count, s);
}

}  // namespace bs
