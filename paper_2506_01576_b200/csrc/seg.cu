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
#include <cstdlib>
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

// lb - (segment start) and the hit flag of an in-range query x, from the
// node k (in [S, 2S)) its descent of the D image levels reached
// SMEM: seg points to shared memory (the staged keys), read with plain loads
template <class K, int D, bool SMEM = false>
__device__ __forceinline__ uint32_t seg_finish(const uint32_t* F, const K* __restrict__ seg, uint32_t len, K smin,
                                               uint32_t sh, K x, uint32_t k, bool* hit) {
    constexpr uint32_t S = 1u << D;
    auto rd = [&](uint32_t i) -> K { if constexpr (SMEM) return seg[i]; else return ldg(seg + i); };
    uint32_t c = k - S;                  // keys whose image is below q's: <= lb - seg start
    K v;
    if (sh == 0) {
        // exact image: the successor is the last left turn (slot 0 = segment max)
        v = c < len ? (K)(smin + (K)F[k >> __ffs((int)~k)]) : (K)0;
        // only the segment max (slot 0, outside the tree) can be below q here:
        // the last segment's queries above every key
        if (c < len && v < x) c = len;
    } else {
        v = c < len ? rd(c) : (K)0;
        if (c < len && v < x) {
            // keys sharing q's image: gallop, then bisect (seg[c] < x)
            uint32_t l = c + 1, step = 1, h;
            for (;;) {
                h = l - 1 + step;
                if (h >= len) { h = len; break; }
                if (rd(h) >= x) break;
                l = h + 1;
                step <<= 1;
            }
            while (l < h) {
                const uint32_t mid = (l + h) >> 1;
                if (rd(mid) < x) l = mid + 1;
                else h = mid;
            }
            c = l;
            v = c < len ? rd(c) : (K)0;
        }
    }
    *hit = c < len && v == x;
    return c;
}

template <class K, int D>
__device__ __forceinline__ uint32_t seg_search(const uint32_t* F, const K* __restrict__ seg, uint32_t len, K smin,
                                               uint32_t sh, K x, bool* hit) {
    const uint32_t fx = seg_image(x, smin, sh);
    uint32_t k = 1;
#pragma unroll
    for (int d = 0; d < D; ++d) k = 2u * k + (F[k] < fx ? 1u : 0u);
    return seg_finish<K, D>(F, seg, len, smin, sh, x, k, hit);
}

template <int OB>
__device__ __forceinline__ uint64_t enc(uint64_t lb, bool hit) {
    constexpr uint64_t MISS = 1ull << (8 * OB - 1);
    return hit ? lb : (lb | MISS);
}

// SORTED, few queries per key (m < 8 n): per query a descent of the segment's
// 32-bit image tree (Eytzinger order, D levels) + one candidate read.  DB: two
// segment buffers — segment b+1 is staged into the other buffer while b is
// searched, one barrier per segment instead of two (a warp that finishes
// its queries of b stages b+1 instead of waiting at a barrier)
template <class K, int D, int OB, bool DB>
__global__ void __launch_bounds__(1024, 1)
k_seg_sorted_eytz(const SegParams<K> p) {
    constexpr uint32_t S = 1u << D;
    constexpr uint32_t NBUF = DB ? 2u : 1u;
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* F0 = sm;                                        // [NBUF][S] slot 0: segment max; 1..S-1: Eytzinger
    K* SK0 = reinterpret_cast<K*>(sm + NBUF * S);             // [NBUF][S] the segment's keys (the candidate reads)
    uint64_t* bnd = reinterpret_cast<uint64_t*>(SK0 + NBUF * S);   // query ranges of this CTA's segments
    const uint64_t G = gridDim.x, B = p.B, n = p.n, m = p.m;
    const uint64_t b0 = B * blockIdx.x / G, b1 = B * (blockIdx.x + 1) / G;
    const uint32_t nb = (uint32_t)(b1 - b0);
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();

    for (uint32_t i = threadIdx.x; i <= nb; i += blockDim.x) {
        const uint64_t b = b0 + i;
        bnd[i] = b == 0 ? 0 : b >= B ? m : upper_bound_any(p.q, m, ldg(p.a + b * S - 1));
    }
    // the next segment's keys are in flight (registers) while this segment is
    // searched; each thread carries R lookups through the image levels together
    constexpr uint32_t KPT = S / 1024;   // keys per thread (blockDim 1024)
    constexpr uint32_t R = 4;
    K nk[KPT];
    auto load_keys = [&](uint64_t b) {
        const uint64_t lo = b * S;
        const uint32_t len = b < b1 ? (uint32_t)((n - lo) < S ? (n - lo) : S) : 0u;
#pragma unroll
        for (uint32_t k = 0; k < KPT; ++k) {
            const uint32_t i = k * 1024u + threadIdx.x;
            nk[k] = i < len ? ldg(p.a + lo + i) : (K)0;
        }
    };
    // segment b's image and keys from the registers into buffer `buf`
    auto stage = [&](uint32_t buf, uint64_t b, const K* kk) {
        const uint64_t lo = b * S;
        const uint32_t len = (uint32_t)((n - lo) < S ? (n - lo) : S);
        const K smin = ldg(p.a + lo), smax = ldg(p.a + lo + len - 1);
        const uint32_t sh = image_shift(smin, smax);
        uint32_t* F = F0 + buf * S;
        K* SK = SK0 + buf * S;
#pragma unroll
        for (uint32_t k = 0; k < KPT; ++k) {
            const uint32_t i = k * 1024u + threadIdx.x;
            const uint32_t f = i < len ? seg_image(kk[k], smin, sh) : 0xFFFFFFFFu;
            F[i == S - 1 ? 0u : eytz_slot<D>(i)] = f;
            SK[i] = kk[k];
        }
    };
    load_keys(b0);
    if constexpr (DB) {
        if (b0 < b1) {
            K kk[KPT];
#pragma unroll
            for (uint32_t k = 0; k < KPT; ++k) kk[k] = nk[k];
            load_keys(b0 + 1);
            stage(0, b0, kk);
        }
        __syncthreads();   // segment b0 staged (and bnd written)
    }
    for (uint64_t b = b0; b < b1; ++b) {
        const uint64_t lo = b * S;
        const uint32_t len = (uint32_t)((n - lo) < S ? (n - lo) : S);
        const K smin = ldg(p.a + lo), smax = ldg(p.a + lo + len - 1);
        const uint32_t sh = image_shift(smin, smax);
        const uint32_t cur = DB ? (uint32_t)((b - b0) & 1u) : 0u;
        if constexpr (DB) {
            if (b + 1 < b1) {
                // the other buffer was last read for segment b-1, before the barrier
                K kk[KPT];
#pragma unroll
                for (uint32_t k = 0; k < KPT; ++k) kk[k] = nk[k];
                load_keys(b + 2);
                stage(cur ^ 1u, b + 1, kk);
            }
        } else {
            K kk[KPT];
#pragma unroll
            for (uint32_t k = 0; k < KPT; ++k) kk[k] = nk[k];
            load_keys(b + 1);
            __syncthreads();   // previous segment's searches are done with F (and bnd is written)
            stage(0, b, kk);
            __syncthreads();
        }
        const uint32_t* F = F0 + cur * S;
        const K* SK = SK0 + cur * S;
        const K lower = b ? ldg(p.a + lo - 1) : (K)0;
        const bool first = b == 0, last = b == B - 1;
        const uint64_t q0 = bnd[b - b0], q1 = bnd[b - b0 + 1];
        // the descent runs on the shared address a = sb + 4k: a' = 2a - sb + 4 [F[k] < q]
        const uint32_t sb = smem_u32(F);
        const uint32_t step_lt = 4u - sb, step_ge = 0u - sb;
        for (uint64_t i = q0 + threadIdx.x; i < q1; i += 1024u * R) {
            K x[R];
            uint32_t fx[R], kq[R];
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) {
                const uint64_t ir = i + r * 1024u;
                x[r] = ir < q1 ? load_stream(p.q + ir, true, pol_stream) : smin;
                fx[r] = seg_image(x[r], smin, sh);
                kq[r] = sb + 4u;
            }
#pragma unroll
            for (int d = 0; d < D; ++d) {
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    const uint32_t h = lds_u32(kq[r]);
                    kq[r] = 2u * kq[r] + (h < fx[r] ? step_lt : step_ge);
                }
            }
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) kq[r] = (kq[r] - sb) >> 2;
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) {
                const uint64_t ir = i + r * 1024u;
                if (ir >= q1) continue;
                uint64_t lb;
                bool hit;
                if ((first || x[r] > lower) && (last || x[r] <= smax)) {
                    lb = lo + seg_finish<K, D, true>(F, SK, len, smin, sh, x[r], kq[r], &hit);
                } else {
                    // outside the segment's key range (an unsorted batch): plain bisection
                    lb = lower_bound_global(p.a, n, x[r]);
                    hit = lb < n && ldg(p.a + lb) == x[r];
                }
                const uint64_t res = enc<OB>(lb, hit);
                if constexpr (OB == 8) store_stream((uint64_t*)p.out + ir, res, true, pol_stream);
                else store_stream((uint32_t*)p.out + ir, (uint32_t)res, true, pol_stream);
            }
        }
        if constexpr (DB) __syncthreads();   // b+1 staged; every search of b is done with buffer cur
    }
}

// #(c < h : k[c] < x) over a sorted run in shared memory, starting from the
// bracket [l, h] that holds the answer
template <class K>
__device__ __forceinline__ uint32_t smem_lower_bound(const K* k, uint32_t l, uint32_t h, K x) {
    while (l < h) {
        const uint32_t mid = (l + h) >> 1;
        if (k[mid] < x) l = mid + 1;
        else h = mid;
    }
    return l;
}

// SORTED.  Per segment the CTA stages the segment's keys in shared memory
// (two buffers filled by TMA bulk copies: segment b+1 lands while b is
// searched, one barrier per segment).  The segment's queries, in blocks of 32,
// are split evenly over the 32 warps.  Per round of up to 31 blocks, lane l
// finds the exact position of block l's first query by bisection over the
// staged keys (lane 31 of a full round: the next block's) — one bisection per
// 32 queries; then every query of block j that lies between block j's and
// block j+1's first queries (always, for an ordered batch) bisects only the
// bracket between their positions (~log2(32 n / m) steps, the same for the
// whole warp).  A query outside its bracket or its segment's key range (an
// unordered batch) takes a plain bisection of the segment or of the array:
// correct in any order, fast when ordered.
constexpr uint32_t kSegInFlight = 8;   // blocks of 32 queries loaded ahead per warp

template <class K, int D, int OB>
__global__ void __launch_bounds__(1024, 1)
k_seg_sorted(const SegParams<K> p) {
    constexpr uint32_t S = 1u << D;
    extern __shared__ __align__(16) uint32_t sm[];
    K* SK0 = reinterpret_cast<K*>(sm);                          // [2][S] the segment's keys
    uint64_t* bnd = reinterpret_cast<uint64_t*>(SK0 + 2 * S);   // query ranges of this CTA's segments
    const uint64_t G = gridDim.x, B = p.B, n = p.n, m = p.m;
    const uint64_t b0 = B * blockIdx.x / G, b1 = B * (blockIdx.x + 1) / G;
    const uint32_t nb = (uint32_t)(b1 - b0);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();

    uint64_t* bar = bnd + nb + 1;   // [2] one mbarrier per buffer
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    for (uint32_t i = threadIdx.x; i <= nb; i += blockDim.x) {
        const uint64_t b = b0 + i;
        bnd[i] = b == 0 ? 0 : b >= B ? m : upper_bound_any(p.q, m, ldg(p.a + b * S - 1));
    }
    // segment b's keys into buffer buf: a TMA bulk copy issued by thread 0,
    // completed on the buffer's mbarrier (no registers held, the copy overlaps
    // the search of the other buffer); a byte count that is not a multiple of
    // 16 (only the array's last segment) is copied by all threads instead
    auto seg_len = [&](uint64_t b) -> uint32_t {
        const uint64_t lo = b * S;
        return (uint32_t)((n - lo) < S ? (n - lo) : S);
    };
    const bool a16 = ((uintptr_t)p.a & 15u) == 0u;
    auto bulk_ok = [&](uint64_t b) { return a16 && (seg_len(b) * (uint32_t)sizeof(K)) % 16u == 0u; };
    auto stage = [&](uint32_t buf, uint64_t b) {
        K* dst = SK0 + buf * S;
        const K* src = p.a + b * S;
        const uint32_t len = seg_len(b);
        if (bulk_ok(b)) {
            if (threadIdx.x == 0) {
                const uint32_t bytes = len * (uint32_t)sizeof(K);
                mbar_arrive_expect_tx(&bar[buf], bytes);
                for (uint32_t o = 0; o < bytes; o += 32768u)
                    bulk_g2s((char*)dst + o, (const char*)src + o, bytes - o < 32768u ? bytes - o : 32768u, &bar[buf]);
            }
        } else {
            for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) dst[i] = ldg(src + i);
        }
    };
    __syncthreads();   // mbarriers initialised, bnd written
    if (b0 < b1) stage(0, b0);
    __syncthreads();   // a plain-copied first segment is visible
    for (uint64_t b = b0; b < b1; ++b) {
        const uint32_t cur = (uint32_t)((b - b0) & 1u);
        // the other buffer was last read for segment b-1, before the barrier
        if (b + 1 < b1) stage(cur ^ 1u, b + 1);
        // buffer cur's ((b - b0) >> 1)-th fill (a plain-copied segment is the array's
        // last, so no bulk fill of its buffer follows)
        if (bulk_ok(b)) mbar_wait(&bar[cur], (uint32_t)(((b - b0) >> 1) & 1u));
        const K* SK = SK0 + cur * S;
        const uint64_t lo = b * S;
        const uint32_t len = (uint32_t)((n - lo) < S ? (n - lo) : S);
        const K smax = SK[len - 1];
        const K lower = b ? ldg(p.a + lo - 1) : (K)0;
        const bool first = b == 0, last = b == B - 1;
        const uint64_t q0 = bnd[b - b0], q1 = bnd[b - b0 + 1];
        // the segment's blocks of 32 queries, split evenly over the 32 warps
        const uint32_t nblk = (uint32_t)((q1 - q0 + 31) / 32);
        const uint32_t bw0 = (uint32_t)((uint64_t)nblk * warp / 32), bw1 = (uint32_t)((uint64_t)nblk * (warp + 1) / 32);
        for (uint32_t bs = bw0; bs < bw1; bs += 31) {
            const uint32_t nr = (bw1 - bs) < 31u ? (bw1 - bs) : 31u;   // blocks this round
            // splitters: lane l <= nr takes the first query of block bs + l (lane nr:
            // the block after the round) and finds its position by bisection
            const uint64_t si = q0 + 32ull * (bs + lane);
            const bool shas = lane <= nr && si < q1;
            const K sx = shas ? ldg(p.q + si) : (K)0;
            const uint32_t sc = shas ? smem_lower_bound(SK, 0u, len, sx) : len;
            for (uint32_t j0 = 0; j0 < nr; j0 += kSegInFlight) {
                K xs[kSegInFlight];   // kSegInFlight blocks of queries in flight
#pragma unroll
                for (uint32_t u = 0; u < kSegInFlight; ++u) {
                    const uint64_t ir = q0 + 32ull * (bs + j0 + u) + lane;
                    xs[u] = (j0 + u < nr && ir < q1) ? load_stream(p.q + ir, true, pol_stream) : (K)0;
                }
#pragma unroll
                for (uint32_t u = 0; u < kSegInFlight; ++u) {
                    const uint32_t j = j0 + u;
                    if (j >= nr) break;                              // warp-uniform
                    const uint64_t ir = q0 + 32ull * (bs + j) + lane;
                    const K sj = __shfl_sync(0xFFFFFFFFu, sx, j), sj1 = __shfl_sync(0xFFFFFFFFu, sx, j + 1);
                    const uint32_t cl = __shfl_sync(0xFFFFFFFFu, sc, j), ch1 = __shfl_sync(0xFFFFFFFFu, sc, j + 1);
                    const bool has1 = q0 + 32ull * (bs + j + 1) < q1;   // the next block exists
                    const bool valid = ir < q1;
                    const K x = valid ? xs[u] : sj;
                    const bool inseg = (first || x > lower) && (last || x <= smax);
                    const bool inbr = inseg && x >= sj && (!has1 || x <= sj1);
                    // the bracket [cl, ch1] (shared by the warp); lanes outside it take [0, len]
                    const uint32_t c = smem_lower_bound(SK, inbr ? cl : 0u, inbr ? ch1 : len, x);
                    uint64_t lb;
                    bool hit;
                    if (inseg) {
                        lb = lo + c;
                        hit = c < len && SK[c] == x;
                    } else {
                        // outside the segment's key range (an unordered batch): the whole array
                        lb = lower_bound_global(p.a, n, x);
                        hit = lb < n && ldg(p.a + lb) == x;
                    }
                    if (valid) {
                        const uint64_t res = enc<OB>(lb, hit);
                        if constexpr (OB == 8) store_stream((uint64_t*)p.out + ir, res, true, pol_stream);
                        else store_stream((uint32_t*)p.out + ir, (uint32_t)res, true, pol_stream);
                    }
                }
            }
        }
        __syncthreads();   // b+1 staged; every search of b is done with its buffer
    }
}

// ---------------------------------------------------------------- GLOBAL mode

constexpr int kSegLog2 = 13;           // SORTED: S = 8192 keys per segment (a 32-KB image)
constexpr int kGlobLog2 = 15;          // GLOBAL: S = 32768 keys per bucket segment (a 128-KB image)
constexpr uint32_t kPartTile = 8192;   // queries per partition tile (u16 positions)
constexpr uint32_t kGlobMaxB = 2048;   // buckets (n <= 2^26 keys): per-bucket counters fit shared memory
constexpr uint32_t kPartBins = 8192;   // radix directory over the 31-bit maxima images
constexpr uint32_t kPartBinShift = 18; // 2^31 >> 18 = kPartBins

// Slab layout: bucket b's region holds one slab of `cap` queries per partition
// CTA c (slab(b, c) = (b * G + c) * cap), filled in tile order by that CTA
// alone — no global atomics, and each CTA keeps only one partly written line
// per bucket open in L2 (B x G lines, 39 MB at config 3).
template <class K>
struct PartParams {
    const K* a;
    uint64_t n, m;
    const K* q;
    void* out;
    uint32_t B;               // buckets (segments of 2^kGlobLog2 keys)
    uint32_t DB;              // log2 of the maxima tree size (2^DB >= B)
    uint32_t G;               // partition CTAs (tile t belongs to CTA t % G)
    uint32_t cap;             // queries per slab (<= 65535)
    K* rec;                   // [B * G * cap] queries, bucket-major, slab per CTA
    void* res;                // [B * G * cap] their results (same positions)
    uint16_t* slot2;          // [m] tile slot of the tile's j-th query in bucket order
    uint16_t* b2;             // [m] its bucket
    uint16_t* toff;           // [ntiles * B] start of bucket b's run in tile t's bucket order
    uint16_t* tlim;           // [ntiles * B] length of that run stored in the slab (the rest overflowed)
    uint16_t* tstart;         // [ntiles * B] position of tile t's run in slab(b, t % G)
    uint32_t* slabcnt;        // [G * B] queries stored per slab
    uint32_t* ovf_n;          // overflowed queries (slab full: a skewed batch)
    K* ovf_q;                 // [m]
    uint32_t* ovf_j;          // [m] their tile-sorted position t * T + j
    void* res_full;           // [m] results of overflowed queries at t * T + j
    uint32_t stream_hint;
};

// exact bucket from the image bound c: step over maxima still < x (galloping;
// only when the successor's image ties q's — max_c = a[(c+1)*S - 1], c < B-1)
template <class K, int D>
__device__ __forceinline__ uint32_t bucket_fix(const K* __restrict__ a, uint32_t nm, uint32_t c, K x) {
    constexpr uint64_t S = 1ull << D;
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

// block-wide exclusive scan of cnt[0..N) in place (blockDim.x a multiple of 32, <= 1024)
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
        const uint32_t v = lane < (blockDim.x >> 5) ? warp_tmp[lane] : 0u;   // any blockDim <= 1024
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

// Partition: per tile of T queries (tile t on CTA t % G), bucket each query, sort
// the tile by bucket in shared memory, write the tile's (slot, bucket) lists in
// that order, and append each bucket's run to the CTA's slab of that bucket.
template <class K, int D>
__global__ void __launch_bounds__(1024, 1)
k_part(const PartParams<K> p) {
    constexpr uint32_t T = kPartTile, E = T / 1024;
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t B = p.B, DB = p.DB, NT = 1u << DB;
    const uint32_t B4 = (B + 3u) & ~3u;                     // per-bucket arrays padded to 16 B
    K* stq = reinterpret_cast<K*>(sm);                      // [T] queries in bucket order
    uint64_t* dptr = reinterpret_cast<uint64_t*>(stq + T);  // [B] rec index of run position 0 (minus off)
    uint32_t* MS = reinterpret_cast<uint32_t*>(dptr + B4);  // [B] maxima images, sorted (MS[B-1] = max)
    uint32_t* hist = MS + B4;                               // [B]
    uint32_t* off = hist + B4;                              // [B] tile offsets
    uint32_t* run = off + B4;                               // [B] running ranks, then the fitting limit
    uint32_t* cur = run + B4;                               // [B] slab fill of this CTA
    uint32_t* warp_tmp = cur + B4;                          // [32]
    uint16_t* BF = reinterpret_cast<uint16_t*>(warp_tmp + 32);    // [kPartBins + 8] bin -> first bucket
    uint16_t* stb = BF + kPartBins + 8;                            // [T] bucket, bucket order (8-B aligned)
    uint16_t* sts = stb + T;                                       // [T] tile slot, bucket order
    constexpr uint64_t S = 1ull << D;
    const K gbase = ldg(p.a), gtop = ldg(p.a + p.n - 1);
    const uint32_t gsh = image_shift(gbase, gtop);
    // bucket b(q) = #(maxima < q): the maxima's order-preserving images, sorted,
    // and a radix directory over the images' top bits (the partition is one
    // radix-style pass over key ranges): bin x of image f = f >> kPartBinShift
    // holds the buckets [BF[x], BF[x+1]], usually one compare
    for (uint32_t i = threadIdx.x; i < B; i += blockDim.x)
        MS[i] = i + 1 < B ? seg_image(ldg(p.a + ((uint64_t)i + 1) * S - 1), gbase, gsh) : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t x = threadIdx.x; x <= kPartBins + 1; x += blockDim.x) {
        const uint64_t f = (uint64_t)x << kPartBinShift;   // first image of bin x
        uint32_t lo = 0, hi = B - 1;                       // #(MS[c] < f) over the B-1 real maxima
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((uint64_t)MS[mid] < f) lo = mid + 1;
            else hi = mid;
        }
        BF[x] = (uint16_t)lo;
    }
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) cur[b] = 0;
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t ntiles = (p.m + T - 1) / T;
    const uint32_t c = blockIdx.x, G = p.G;
    // the next tile's queries are loaded while this tile is sorted and written
    K xn[E];
    auto load_tile = [&](uint64_t t, K* xs) {
        const uint64_t b0 = t * T;
        const K* qp = p.q + b0 + threadIdx.x;
        if (b0 + T <= p.m) {
#pragma unroll
            for (uint32_t e = 0; e < E; ++e) xs[e] = load_stream(qp + e * 1024u, true, pol_stream);
        } else {
#pragma unroll
            for (uint32_t e = 0; e < E; ++e)
                xs[e] = (b0 + e * 1024u + threadIdx.x < p.m) ? load_stream(qp + e * 1024u, true, pol_stream) : (K)0;
        }
    };
    load_tile(c, xn);
    for (uint64_t t = c; t < ntiles; t += G) {
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) { hist[b] = 0; run[b] = 0; }
        __syncthreads();   // (also: the maxima image and cur are ready)
        K x[E];
        uint32_t bk[E];
        const uint64_t base = t * T;
        const uint32_t cnt = (uint32_t)((p.m - base) < T ? (p.m - base) : T);
        uint32_t fx[E], lo[E], hi[E];
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) x[e] = xn[e];
        if (t + G < ntiles) load_tile(t + G, xn);
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            fx[e] = seg_image(x[e], gbase, gsh);
            const uint32_t bin = fx[e] >> kPartBinShift;
            lo[e] = BF[bin];
            hi[e] = BF[bin + 1];
        }
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            const uint32_t j = e * 1024u + threadIdx.x;
            bk[e] = 0xFFFFFFFFu;
            if (j < cnt) {
                // #(maxima with image < fx) lies in [lo, hi]: step (bisect when the bin is crowded)
                uint32_t l = lo[e], h = hi[e];
                while (h - l > 4) {
                    const uint32_t mid = (l + h) >> 1;
                    if (MS[mid] < fx[e]) l = mid + 1;
                    else h = mid;
                }
                while (l < h && MS[l] < fx[e]) ++l;
                uint32_t b = l;
                if (b < B - 1 && MS[b] == fx[e]) b = bucket_fix<K, D>(p.a, B - 1, b, x[e]);
                bk[e] = b;
                atomicAdd(&hist[b], 1u);
            }
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) off[b] = hist[b];
        __syncthreads();
        block_exscan(off, B, warp_tmp);
        // tile meta for the unpartition: run start, stored length and slab position per bucket
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) {
            const uint32_t room = p.cap - cur[b];
            p.toff[t * B + b] = (uint16_t)off[b];
            p.tlim[t * B + b] = (uint16_t)(hist[b] < room ? hist[b] : room);
            p.tstart[t * B + b] = (uint16_t)cur[b];
        }
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            if (bk[e] == 0xFFFFFFFFu) continue;
            const uint32_t pos = off[bk[e]] + atomicAdd(&run[bk[e]], 1u);
            stq[pos] = x[e];
            stb[pos] = (uint16_t)bk[e];
            sts[pos] = (uint16_t)(e * 1024u + threadIdx.x);
        }
        __syncthreads();
        // per bucket: where run position j lands in the slab, and how much of the run fits
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) {
            dptr[b] = ((uint64_t)b * G + c) * p.cap + cur[b] - off[b];
            run[b] = off[b] + (p.cap - cur[b]);
        }
        // the tile's (slot, bucket) lists in bucket order: 8-B vector copies
        for (uint32_t j4 = threadIdx.x * 4; j4 < cnt; j4 += blockDim.x * 4) {
            if (j4 + 4 <= cnt) {
                *reinterpret_cast<uint2*>(p.slot2 + base + j4) = *reinterpret_cast<const uint2*>(sts + j4);
                *reinterpret_cast<uint2*>(p.b2 + base + j4) = *reinterpret_cast<const uint2*>(stb + j4);
            } else {
                for (uint32_t j = j4; j < cnt; ++j) { p.slot2[base + j] = sts[j]; p.b2[base + j] = stb[j]; }
            }
        }
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
            const uint32_t b = stb[j];
            const K xq = stq[j];
            if (j < run[b]) {
                p.rec[dptr[b] + j] = xq;
            } else {
                const uint32_t o = atomicAdd(p.ovf_n, 1u);
                p.ovf_q[o] = xq;
                p.ovf_j[o] = (uint32_t)(base + j);
            }
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) {
            const uint32_t v = cur[b] + hist[b];
            cur[b] = v < p.cap ? v : p.cap;
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) p.slabcnt[(uint64_t)c * B + b] = cur[b];
}

// Segment lookups per bucket: the bucket's G slabs, results at the same positions.
template <class K, int D, int OB>
__global__ void __launch_bounds__(1024, 1)
k_seg_part(const PartParams<K> p) {
    using O = typename std::conditional<OB == 8, uint64_t, uint32_t>::type;
    constexpr uint32_t S = 1u << D;
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* F = sm;
    const uint64_t GC = gridDim.x, B = p.B, n = p.n;
    // work items: bucket b split into P parts of its slabs (P > 1 only when there
    // are fewer buckets than twice the CTAs); consecutive items share a segment
    const uint64_t P = B >= 2 * GC ? 1 : (2 * GC + B - 1) / B;
    const uint64_t I = B * P;
    const uint64_t i0 = I * blockIdx.x / GC, i1 = I * (blockIdx.x + 1) / GC;
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
        const uint32_t c0 = (uint32_t)(p.G * part / P), c1 = (uint32_t)(p.G * (part + 1) / P);
        // one warp per slab; R queries per lane descend together (their
        // shared-memory and global latencies overlap)
        constexpr uint32_t R = 4;
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (uint32_t c = c0 + warp; c < c1; c += nw) {
            const uint64_t sb = ((uint64_t)b * p.G + c) * p.cap;
            const uint32_t cnt = p.slabcnt[(uint64_t)c * B + b];
            for (uint32_t j0 = 0; j0 < cnt; j0 += 32 * R) {
                K x[R];
                uint32_t k[R], fx[R];
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    const uint32_t j = j0 + r * 32 + lane;
                    x[r] = j < cnt ? p.rec[sb + j] : smin;
                    fx[r] = seg_image(x[r], smin, sh);
                    k[r] = 1;
                }
#pragma unroll
                for (int d = 0; d < D; ++d) {
#pragma unroll
                    for (uint32_t r = 0; r < R; ++r) k[r] = 2u * k[r] + (F[k[r]] < fx[r] ? 1u : 0u);
                }
                uint32_t cc[R];
                K v[R];
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    cc[r] = k[r] - S;
                    if (sh == 0) v[r] = cc[r] < len ? (K)(smin + (K)F[k[r] >> __ffs((int)~k[r])]) : (K)0;
                    else v[r] = cc[r] < len ? ldg(seg + cc[r]) : (K)0;
                }
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    const uint32_t j = j0 + r * 32 + lane;
                    if (j >= cnt) continue;
                    uint32_t c2 = cc[r];
                    K vv = v[r];
                    if (c2 < len && vv < x[r]) {
                        if (sh == 0) {
                            c2 = len;   // only the segment max (slot 0) can be below q
                        } else {
                            bool h;
                            c2 = seg_search<K, D>(F, seg, len, smin, sh, x[r], &h);
                            vv = c2 < len ? ldg(seg + c2) : (K)0;
                        }
                    }
                    const bool hit = c2 < len && vv == x[r];
                    ((O*)p.res)[sb + j] = (O)enc<OB>(lo + c2, hit);
                }
            }
        }
    }
}

template <class K, int OB>
__global__ void k_part_ovf(const PartParams<K> p) {
    using O = typename std::conditional<OB == 8, uint64_t, uint32_t>::type;
    const uint32_t no = *p.ovf_n;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < no; j += (uint64_t)gridDim.x * blockDim.x) {
        const K x = p.ovf_q[j];
        const uint64_t lb = lower_bound_global(p.a, p.n, x);
        const bool hit = lb < p.n && ldg(p.a + lb) == x;
        ((O*)p.res_full)[p.ovf_j[j]] = (O)enc<OB>(lb, hit);
    }
}

// Unpartition: per tile (on CTA t % G, in the partition's tile order, so each
// slab line is read while L2 still holds it) gather the tile's results run by
// run, scatter them to query order in shared memory, one coalesced store.
constexpr uint32_t kUnpartThreads = 1024;

// Unpartition: per tile (tile t's runs sit in the slabs of owner t % G) gather
// the tile's results run by run, scatter them to query order in shared memory,
// store the tile coalesced.  The next tile's meta (run start, stored length,
// slab position per bucket) and its (bucket, slot) lists are loaded while this
// tile is gathered.
template <class K, int OB>
__global__ void __launch_bounds__(kUnpartThreads, 1)
k_unpart(const PartParams<K> p) {
    using O = typename std::conditional<OB == 8, uint64_t, uint32_t>::type;
    constexpr uint32_t T = kPartTile, E = T / kUnpartThreads;
    constexpr uint32_t MB = kGlobMaxB / kUnpartThreads;   // meta entries per thread
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t B = p.B, G = p.G;
    O* tile = reinterpret_cast<O*>(sm);                      // [T]
    uint32_t* off = reinterpret_cast<uint32_t*>(tile + T);   // [B] run start in the tile's bucket order
    uint32_t* src = off + B;                                 // [B] run start in the slab
    uint32_t* lim = src + B;                                 // [B] stored run length
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t ntiles = (p.m + T - 1) / T;
    uint32_t no[MB], ns[MB], nl[MB], nb[E], nsl[E];
    auto prefetch = [&](uint64_t t) {
        const uint64_t base = t * T;
        const uint32_t cnt = (uint32_t)((p.m - base) < T ? (p.m - base) : T);
#pragma unroll
        for (uint32_t i = 0; i < MB; ++i) {
            const uint32_t b = i * kUnpartThreads + threadIdx.x;
            if (b < B) {
                no[i] = p.toff[t * B + b];
                nl[i] = p.tlim[t * B + b];
                ns[i] = p.tstart[t * B + b];
            }
        }
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            const uint32_t j = e * kUnpartThreads + threadIdx.x;
            nb[e] = j < cnt ? p.b2[base + j] : 0u;
            nsl[e] = j < cnt ? p.slot2[base + j] : 0u;
        }
    };
    if (blockIdx.x < ntiles) prefetch(blockIdx.x);
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t base = t * T;
        const uint32_t cnt = (uint32_t)((p.m - base) < T ? (p.m - base) : T);
        const uint32_t c = (uint32_t)(t % G);
#pragma unroll
        for (uint32_t i = 0; i < MB; ++i) {
            const uint32_t b = i * kUnpartThreads + threadIdx.x;
            if (b < B) { off[b] = no[i]; src[b] = ns[i]; lim[b] = nl[i]; }
        }
        uint32_t bb[E], sl[E];
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) { bb[e] = nb[e]; sl[e] = nsl[e]; }
        if (t + gridDim.x < ntiles) prefetch(t + gridDim.x);
        __syncthreads();
        O v[E];
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            const uint32_t j = e * kUnpartThreads + threadIdx.x;
            if (j < cnt) {
                const uint32_t b = bb[e], r = j - off[b];
                const O* sp = r < lim[b] ? (const O*)p.res + (((uint64_t)b * G + c) * p.cap + src[b] + r)
                                         : (const O*)p.res_full + (base + j);
                v[e] = *sp;
            }
        }
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            const uint32_t j = e * kUnpartThreads + threadIdx.x;
            if (j < cnt) tile[sl[e]] = v[e];
        }
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x)
            store_stream((O*)p.out + base + j, tile[j], true, pol_stream);
    }
}

// ---------------------------------------------------------------- launchers

// two buffers of one segment's keys + the per-segment query ranges
static uint64_t seg_smem_bytes(uint64_t n, uint32_t grid, uint32_t kb) {
    const uint64_t S = 1ull << kSegLog2;
    const uint64_t B = (n + S - 1) / S;
    const uint64_t nb = (B + grid - 1) / grid + 1;
    return 2 * S * kb + nb * 8 + 16;
}
constexpr uint64_t kSegSmemMax = 200u * 1024u;

template <class K, int D, int OB>
static cudaError_t go_seg(const SegParams<K>& p, Grid grid, cudaStream_t s, bool* uns) {
    auto kern = k_seg_sorted<K, D, OB>;
    const uint32_t threads = 1024;
    uint64_t g = 0;
    grid.sched_static = 1;
    grid.ctas_per_sm = 1;
    const uint32_t smem = (uint32_t)seg_smem_bytes(p.n, grid.sm_count, (uint32_t)sizeof(K));
    cudaError_t e = plan_grid((const void*)kern, threads, smem, grid, grid.sm_count, carveout_for(smem, threads), &g, uns);
    if (e != cudaSuccess || *uns) return e;
    kern<<<(unsigned)g, threads, smem, s>>>(p);
    count_launch();
    return cudaGetLastError();
}

static uint64_t seg_smem_bytes_eytz(uint64_t n, uint32_t grid, uint32_t kb, uint32_t nbuf = 1) {
    const uint64_t S = 1ull << kSegLog2;
    const uint64_t B = (n + S - 1) / S;
    const uint64_t nb = (B + grid - 1) / grid + 1;
    return nbuf * S * (4 + kb) + nb * 8 + 16;
}

template <class K, int D, int OB>
static cudaError_t go_seg_eytz(const SegParams<K>& p, Grid grid, cudaStream_t s, bool* uns) {
    // two segment buffers when they fit (DB), else one
    const bool db = seg_smem_bytes_eytz(p.n, grid.sm_count, (uint32_t)sizeof(K), 2) <= kSegSmemMax;
    auto kern = db ? k_seg_sorted_eytz<K, D, OB, true> : k_seg_sorted_eytz<K, D, OB, false>;
    const uint32_t threads = 1024;
    uint64_t g = 0;
    grid.sched_static = 1;
    grid.ctas_per_sm = 1;
    const uint32_t smem = (uint32_t)seg_smem_bytes_eytz(p.n, grid.sm_count, (uint32_t)sizeof(K), db ? 2u : 1u);
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
    // bracketed bisection over the staged keys for u32 keys, and for u64 keys
    // with many queries per key (m >= 32 n: a block of 32 queries brackets ~1
    // key); otherwise the image-tree descent, whose fixed D levels of 32-bit
    // probes cost less than a 64-bit bisection of a wide bracket (measured,
    // DESIGN.md §6.9, profiles/r2s3/seg_kernel_ab.jsonl).  BS_SEG_KERNEL=
    // eytz|bracket forces one (A/B).
    bool bracket = kb == 4 || m >= 32 * n;
    if (const char* v = getenv("BS_SEG_KERNEL")) bracket = strcmp(v, "bracket") == 0 ? true : strcmp(v, "eytz") == 0 ? false : bracket;
    if (bracket ? seg_smem_bytes(n, grid.sm_count, (uint32_t)kb) > kSegSmemMax
                : seg_smem_bytes_eytz(n, grid.sm_count, (uint32_t)kb) > kSegSmemMax) {
        *uns = true;
        return cudaSuccess;
    }
    if (kb == 8) {
        SegParams<uint64_t> p{(const uint64_t*)a, n, (const uint64_t*)q, m, out, (uint32_t)ob, (n + S - 1) / S, stream_hint};
        if (bracket) return ob == 8 ? go_seg<uint64_t, D, 8>(p, grid, s, uns) : go_seg<uint64_t, D, 4>(p, grid, s, uns);
        return ob == 8 ? go_seg_eytz<uint64_t, D, 8>(p, grid, s, uns) : go_seg_eytz<uint64_t, D, 4>(p, grid, s, uns);
    }
    SegParams<uint32_t> p{(const uint32_t*)a, n, (const uint32_t*)q, m, out, (uint32_t)ob, (n + S - 1) / S, stream_hint};
    if (bracket) return ob == 8 ? go_seg<uint32_t, D, 8>(p, grid, s, uns) : go_seg<uint32_t, D, 4>(p, grid, s, uns);
    return ob == 8 ? go_seg_eytz<uint32_t, D, 8>(p, grid, s, uns) : go_seg_eytz<uint32_t, D, 4>(p, grid, s, uns);
}

// workspace layout of the GLOBAL mode (all offsets 256-B aligned)
struct PartLayout {
    uint64_t B, G, cap, ntiles;
    uint64_t o_rec, o_res, o_slot2, o_b2, o_toff, o_tlim, o_tstart, o_slabcnt, o_ovfn, o_ovfq, o_ovfj, o_resfull, total;
};

static uint64_t al256(uint64_t x) { return (x + 255) & ~255ull; }

static bool part_layout(uint64_t n, uint64_t m, int kb, int ob, uint32_t G, PartLayout* L) {
    const uint64_t S = 1ull << kGlobLog2;
    L->B = (n + S - 1) / S;
    L->G = G;
    if (L->B > kGlobMaxB || m >= (1ull << 32)) return false;
    const uint64_t mm = m ? m : 1;
    L->ntiles = (mm + kPartTile - 1) / kPartTile;
    uint64_t cap = (mm + L->B * G - 1) / (L->B * G);   // expected queries per slab
    cap += cap / 4 + 64;                                 // + slack (beyond: the overflow list)
    if (cap > 65535) cap = 65535;
    L->cap = cap;
    const uint64_t slots = L->B * G * cap;
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) { const uint64_t r = o; o += al256(bytes); return r; };
    L->o_rec = take(slots * kb);
    L->o_res = take(slots * ob);
    L->o_slot2 = take(2 * mm);
    L->o_b2 = take(2 * mm);
    L->o_toff = take(2 * L->ntiles * L->B);
    L->o_tlim = take(2 * L->ntiles * L->B);
    L->o_tstart = take(2 * L->ntiles * L->B);
    L->o_slabcnt = take(4 * G * L->B);
    L->o_ovfn = take(4);
    L->o_ovfq = take(kb * mm);
    L->o_ovfj = take(4 * mm);
    L->o_resfull = take((uint64_t)ob * mm);
    L->total = o;
    return true;
}

bool part_workspace_bytes(uint64_t n, uint64_t m, int kb, int ob, uint32_t sm_count, uint64_t* bytes) {
    PartLayout L;
    if (!part_layout(n, m, kb, ob, sm_count, &L)) return false;
    *bytes = L.total;
    return true;
}

template <class K, int OB>
static cudaError_t go_part(PartParams<K> p, const PartLayout& L, char* ws, uint32_t sm_count, cudaStream_t s) {
    constexpr int D = kGlobLog2;
    p.B = (uint32_t)L.B;
    p.G = (uint32_t)L.G;
    p.cap = (uint32_t)L.cap;
    p.rec = (K*)(ws + L.o_rec);
    p.res = ws + L.o_res;
    p.slot2 = (uint16_t*)(ws + L.o_slot2);
    p.b2 = (uint16_t*)(ws + L.o_b2);
    p.toff = (uint16_t*)(ws + L.o_toff);
    p.tlim = (uint16_t*)(ws + L.o_tlim);
    p.tstart = (uint16_t*)(ws + L.o_tstart);
    p.slabcnt = (uint32_t*)(ws + L.o_slabcnt);
    p.ovf_n = (uint32_t*)(ws + L.o_ovfn);
    p.ovf_q = (K*)(ws + L.o_ovfq);
    p.ovf_j = (uint32_t*)(ws + L.o_ovfj);
    p.res_full = ws + L.o_resfull;
    uint32_t lb = 0;
    while ((1ull << lb) < L.B) ++lb;
    p.DB = lb ? lb : 1;
    cudaError_t e = cudaMemsetAsync(p.ovf_n, 0, 4, s);
    if (e != cudaSuccess) return e;
    bool uns = false;
    uint64_t g = 0;
    {   // partition: exactly G CTAs (tile t on CTA t % G; the unpartition relies on it)
        auto kern = k_part<K, D>;
        const uint32_t B4 = (p.B + 3u) & ~3u;
        const uint32_t smem = kPartTile * (uint32_t)sizeof(K) + 8u * B4 + 4u * (5u * B4 + 32u) + 2u * (kPartBins + 8) + 4u * kPartTile;
        Grid grid{1u, 1u, p.G};
        e = plan_grid((const void*)kern, 1024, smem, grid, p.G, carveout_for(smem, 1024), &g, &uns);
        if (e != cudaSuccess) return e;
        if (uns || g != p.G) return cudaErrorInvalidConfiguration;
        kern<<<(unsigned)g, 1024, smem, s>>>(p);
        count_launch();
    }
    {   // segment lookups per bucket
        auto kern = k_seg_part<K, D, OB>;
        const uint32_t smem = 4u << D;
        Grid grid{1u, 1u, sm_count};
        e = plan_grid((const void*)kern, 1024, smem, grid, sm_count, carveout_for(smem, 1024), &g, &uns);
        if (e != cudaSuccess) return e;
        if (uns) return cudaErrorInvalidConfiguration;
        kern<<<(unsigned)g, 1024, smem, s>>>(p);
        count_launch();
    }
    k_part_ovf<K, OB><<<sm_count, 256, 0, s>>>(p);
    count_launch();
    {   // back to query order (slab owner = tile % G is an address, not a CTA)
        auto kern = k_unpart<K, OB>;
        const uint32_t smem = kPartTile * OB + 4u * (3u * p.B);
        Grid grid{1u, 1u, sm_count};
        e = plan_grid((const void*)kern, kUnpartThreads, smem, grid, sm_count, carveout_for(smem, kUnpartThreads),
                      &g, &uns);
        if (e != cudaSuccess) return e;
        if (uns) return cudaErrorInvalidConfiguration;
        kern<<<(unsigned)g, kUnpartThreads, smem, s>>>(p);
        count_launch();
    }
    return cudaGetLastError();
}

cudaError_t launch_part_global(int kb, int ob, const void* a, uint64_t n, const void* q, uint64_t m, void* out,
                               uint32_t stream_hint, void* ws, uint64_t ws_bytes, uint32_t sm_count, cudaStream_t s,
                               bool* uns) {
    PartLayout L;
    if (!part_layout(n, m, kb, ob, sm_count, &L) || ws_bytes < L.total) { *uns = true; return cudaSuccess; }
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
