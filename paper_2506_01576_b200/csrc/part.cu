// part.cu — BS_REORDER_BUCKET: a random batch turned into L2-local work.
//
// PAPER.md §4.3: neighbouring lookups in key order share their
// search paths; the paper sorts lookups locally (per thread block) because a
// global, out-of-place sort of the batch is "too expensive".  On B200 the
// random-order lookup is bound by one random DRAM line per lookup (the DRAM
// atom), so the only way past ~36 G random lines/s is to make
// the array accesses of a batch local in time.  This mode partitions the batch
// by KEY RANGE into buckets whose slice of the array fits L2, searches bucket
// after bucket, and restores query order — a coarse global reorder that costs
// three streaming passes instead of a sort:
//
//   k_bk_hist    per CTA: histogram of its tiles' queries over the B buckets;
//                each query's bucket id is stored for the partition pass
//   k_bk_scan    per bucket: exclusive prefix of the CTA histograms
//   k_bk_part    per tile of T = 8192 queries: rank each query in its bucket's
//                run (shared atomic), counting-sort the tile by bucket in shared
//                memory (query and slot word in one 16-B entry), append each run to the CTA's slice of its bucket's
//                region (bucket-major, exact offsets: no global atomics, no
//                overflow), and record for every sorted position its bucket and
//                original slot
//   k_bk_search  items of queries in bucket order from a global counter: per
//                bucket a pinned Eytzinger table of its 2^D unit maxima (§4.2's
//                pinned top levels of a binary search, built by bs_build) is
//                staged by TMA; each lookup descends D levels in shared memory,
//                then (two-level buckets) reads one 32-B node of leaf-maxima
//                images, then reads its leaf (L2-resident while the bucket is
//                worked on) and counts the keys < q (§5's leaf scan)
//   k_bk_unpart  per tile: gather the results of its runs, scatter them to query
//                order in shared memory, one coalesced store (Listing 2 l.35-39's
//                "unsort", at batch scale)
//
// Peer window (bs_lookup_peer with layout.reorder = BUCKET, peer.cu): the same
// passes over the receive window, the batch size read from the receive cursor
// on the device (the PM kernel variants), and k_bk_unpart storing every result
// into its source rank's return window instead of `out`.
//
// Bucket b covers the array positions [b*NB, (b+1)*NB): fine buckets hold 2^D
// leaves of 32 B (NB = 2^17 u64 / 2^18 u32 keys), two-level buckets 2^D units of
// 16 leaves of 32 B (16 MB of keys; 8 leaves of 64 B with BS_BUCKET_G8=1).  A query belongs to bucket #(bucket maxima <
// q) (the last bucket also takes the queries above every key).  The bucket is
// exact, so the per-bucket search never leaves its bucket.  DESIGN.md §6.11.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "params.h"
#include "peer_sync.cuh"

namespace bs {

constexpr uint32_t kBkTile = 8192;        // queries per partition tile (u16 slots); measured: 4096 (2 CTAs of
                                          // 512 threads per SM) 3.30 ms, 8192 3.08 ms, 16384 3.19 ms at config 3
constexpr uint32_t kBkPThreads = 1024;    // threads of the streaming passes (hist / part / unpart)
constexpr uint32_t kBkUCtas = kBkTile * 8u <= (96u << 10) ? 2u : 1u;   // unpartition CTAs per SM
constexpr uint32_t kBkPCtas = 1;          // their CTAs per SM (tile t on CTA t % (kBkPCtas x SMs));
                                          // measured: 2048-query tiles on 4 CTAs of 256 threads per SM
                                          // halve the runs and cost 30 % more DRAM bytes (4.3 ms)
constexpr uint32_t kBkBinsLog2 = 13;      // radix directory over the 32-bit global image
constexpr uint32_t kBkBins = 1u << kBkBinsLog2;
constexpr uint32_t kBkThreads = 1024;        // threads of the search (one CTA per SM)

// order-preserving 32-bit image of x over [base, ...): 0 at or below base,
// (x - base) >> sh clamped to 2^32 - 1 (exact when the span fits 32 bits)
__device__ __forceinline__ uint32_t bk_img(uint64_t x, uint64_t base, uint32_t sh) {
    if (x <= base) return 0u;
    const uint64_t d = (x - base) >> sh;
    return d > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)d;
}

// shift that makes a span fit 32 bits
__host__ __device__ __forceinline__ uint32_t bk_shift(uint64_t span) {
    uint32_t bl = 0;
    while (bl < 64 && (span >> bl) != 0) ++bl;
    return bl > 32u ? bl - 32u : 0u;
}

// 32 bytes of keys (one sector) without L1 allocation, with an L2 policy
__device__ __forceinline__ void ld_sector(const void* p, uint64_t pol, uint64_t* x) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p), "l"(pol));
}

template <class K>
__device__ __forceinline__ K bk_key(const uint64_t* x, int u) {
    if constexpr (sizeof(K) == 8) return x[u];
    else return (uint32_t)(x[u >> 1] >> (32 * (u & 1)));
}

// ------------------------------------------------------------------ build

// Per bucket b: the Eytzinger table of its leaf maxima images (slot s >= 1
// holds in-order leaf i = (2j+1) 2^(D-1-d) - 1 for s = 2^d + j; slot 0 unused;
// leaves past the array: 0xFFFFFFFF) and its image parameters (base, shift).
template <class K>
__global__ void k_bk_build_tab(const K* __restrict__ a, uint64_t n, uint32_t D, uint32_t LK, uint64_t B,
                               uint32_t* __restrict__ tab, uint64_t* __restrict__ par) {
    const uint64_t S = 1ull << D, NB = S * LK;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= B * S) return;
    const uint64_t b = g >> D, s = g & (S - 1);
    const uint64_t lo = b * NB, len = (n - lo) < NB ? (n - lo) : NB;
    const uint64_t base = (uint64_t)a[lo];
    const uint32_t sh = bk_shift((uint64_t)a[lo + len - 1] - base);
    if (s == 0) {
        par[2 * b] = base;
        par[2 * b + 1] = sh;
        tab[g] = 0;
        return;
    }
    const uint32_t d = 31u - (uint32_t)__clz((int)(uint32_t)s);
    const uint64_t j = s - (1ull << d);
    const uint64_t i = (2 * j + 1) * (1ull << (D - 1 - d)) - 1;   // in-order leaf
    const uint64_t Mb = (len + LK - 1) / LK;
    uint32_t f = 0xFFFFFFFFu;
    if (i < Mb) {
        const uint64_t e = (i + 1) * LK < len ? (i + 1) * LK : len;
        f = bk_img((uint64_t)a[lo + e - 1], base, sh);
    }
    tab[g] = f;
}

// Global images of the bucket maxima (b < B-1; [B-1] = 0xFFFFFFFF) and the
// radix directory dir[x] = #(b < B-1 : max image < x << (32 - kBkBinsLog2)).
template <class K>
__global__ void k_bk_build_dir(const K* __restrict__ a, uint64_t n, uint64_t NB, uint32_t B, uint64_t gbase,
                               uint32_t gsh, uint32_t* __restrict__ mx, uint16_t* __restrict__ dir) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < B) mx[g] = g + 1 < B ? bk_img((uint64_t)a[((uint64_t)g + 1) * NB - 1], gbase, gsh) : 0xFFFFFFFFu;
    if (g <= kBkBins) {
        const uint64_t f = (uint64_t)g << (32 - kBkBinsLog2);
        uint32_t lo = 0, hi = B - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            const uint64_t v = bk_img((uint64_t)a[((uint64_t)mid + 1) * NB - 1], gbase, gsh);
            if (v < f) lo = mid + 1;
            else hi = mid;
        }
        dir[g] = (uint16_t)lo;
    }
}

// Two-level buckets (G > 1): per bucket, the images of all its leaf maxima in
// leaf order (G per table unit, one 32-B node each); leaves past the array:
// 0xFFFFFFFF.  Uses the bucket parameters written by k_bk_build_tab.
template <class K>
__global__ void k_bk_build_gnode(const K* __restrict__ a, uint64_t n, uint32_t D, uint32_t LK, uint32_t G, uint64_t B,
                                 const uint64_t* __restrict__ par, uint32_t* __restrict__ gnode) {
    const uint64_t per = (uint64_t)G << D, NB = per * LK;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= B * per) return;
    const uint64_t b = g / per, i = g % per;
    const uint64_t lo = b * NB, len = (n - lo) < NB ? (n - lo) : NB;
    uint32_t f = 0xFFFFFFFFu;
    if (i * LK < len) {
        const uint64_t e = (i + 1) * LK < len ? (i + 1) * LK : len;
        f = bk_img((uint64_t)a[lo + e - 1], par[2 * b], (uint32_t)par[2 * b + 1]);
    }
    gnode[g] = f;
}

// Two-level buckets with 16-leaf units (G = 16): per unit one 32-B node of 16
// 16-bit images of its leaf maxima, RELATIVE to the unit's image range: with
// lo = image of unit u-1's maximum (0 for u = 0) and hi = image of unit u's
// maximum (2^32 - 1 for the last unit, which the table does not hold), s =
// bitlen(hi - lo) - 16 (>= 0), g = min((image - lo) >> s, 2^16 - 1).  The
// search's descent sees exactly these lo / hi (the last probes below and at or
// above q's image), so the query's g uses the same s.  Leaves past the array:
// 0xFFFF.  Uses the bucket parameters written by k_bk_build_tab.
__device__ __forceinline__ uint32_t bk_sub_shift(uint32_t lo, uint32_t hi) {
    const uint32_t span = hi - lo;
    const uint32_t bl = span ? 32u - (uint32_t)__clz((int)span) : 0u;
    return bl > 16u ? bl - 16u : 0u;
}

template <class K>
__global__ void k_bk_build_gnode16(const K* __restrict__ a, uint64_t n, uint32_t D, uint32_t LK, uint64_t B,
                                   const uint64_t* __restrict__ par, uint16_t* __restrict__ gnode) {
    constexpr uint32_t G = 16;
    const uint64_t per = (uint64_t)G << D, NB = per * LK, S = 1ull << D;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= B * per) return;
    const uint64_t b = g / per, i = g % per, u = i / G;
    const uint64_t lo = b * NB, len = (n - lo) < NB ? (n - lo) : NB;
    const uint64_t base = par[2 * b];
    const uint32_t sh = (uint32_t)par[2 * b + 1];
    auto unit_max_img = [&](uint64_t v) -> uint32_t {   // image of unit v's maximum (0xFFFFFFFF past the keys)
        if (v * G * LK >= len) return 0xFFFFFFFFu;
        const uint64_t e = (v + 1) * G * LK < len ? (v + 1) * G * LK : len;
        return bk_img((uint64_t)a[lo + e - 1], base, sh);
    };
    const uint32_t flo = u == 0 ? 0u : unit_max_img(u - 1);
    const uint32_t fhi = u + 1 == S ? 0xFFFFFFFFu : unit_max_img(u);
    uint16_t r = 0xFFFFu;
    if (i * LK < len) {
        const uint64_t e = (i + 1) * LK < len ? (i + 1) * LK : len;
        const uint32_t f = bk_img((uint64_t)a[lo + e - 1], base, sh);
        const uint32_t d = (f > flo ? f - flo : 0u) >> bk_sub_shift(flo, fhi);
        r = (uint16_t)(d > 0xFFFFu ? 0xFFFFu : d);
    }
    gnode[g] = r;
}

cudaError_t build_bucket_index(int kb, const void* a, uint64_t n, uint32_t D, uint32_t G, uint32_t LB, uint64_t NB,
                               uint64_t B, uint64_t gbase, uint32_t gsh, uint32_t* tab, uint64_t* par, uint32_t* gnode,
                               uint32_t* mx, uint16_t* dir, cudaStream_t s) {
    const uint32_t LK = LB / (uint32_t)kb;   // keys per leaf
    const uint32_t g2 = (uint32_t)(((B > kBkBins + 1 ? B : kBkBins + 1) + 255) / 256);
    if (tab) {
        const uint64_t tot = B << D;
        const uint32_t g1 = (uint32_t)((tot + 255) / 256);
        // table unit = G leaves
        if (kb == 8) k_bk_build_tab<uint64_t><<<g1, 256, 0, s>>>((const uint64_t*)a, n, D, LK * G, B, tab, par);
        else k_bk_build_tab<uint32_t><<<g1, 256, 0, s>>>((const uint32_t*)a, n, D, LK * G, B, tab, par);
        if (G > 1) {
            const uint64_t tn = (B << D) * G;
            const uint32_t g3 = (uint32_t)((tn + 255) / 256);
            uint16_t* g16 = reinterpret_cast<uint16_t*>(gnode);
            if (G == 16 && kb == 8) k_bk_build_gnode16<uint64_t><<<g3, 256, 0, s>>>((const uint64_t*)a, n, D, LK, B, par, g16);
            else if (G == 16) k_bk_build_gnode16<uint32_t><<<g3, 256, 0, s>>>((const uint32_t*)a, n, D, LK, B, par, g16);
            else if (kb == 8) k_bk_build_gnode<uint64_t><<<g3, 256, 0, s>>>((const uint64_t*)a, n, D, LK, G, B, par, gnode);
            else k_bk_build_gnode<uint32_t><<<g3, 256, 0, s>>>((const uint32_t*)a, n, D, LK, G, B, par, gnode);
        }
    }
    if (kb == 8) k_bk_build_dir<uint64_t><<<g2, 256, 0, s>>>((const uint64_t*)a, n, NB, (uint32_t)B, gbase, gsh, mx, dir);
    else k_bk_build_dir<uint32_t><<<g2, 256, 0, s>>>((const uint32_t*)a, n, NB, (uint32_t)B, gbase, gsh, mx, dir);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ lookup

template <class K>
struct BkParams {
    const K* a;
    uint64_t n;
    const K* q;
    uint64_t m;
    void* out;
    uint32_t B;              // buckets
    uint32_t D;              // per-bucket table depth: 2^D units per bucket
    uint32_t LB;             // leaf bytes (32 or 64)
    uint32_t G;              // leaves per unit (1, 8 or 16)
    uint64_t NB;             // keys per bucket = 2^D * LK
    const uint32_t* tab;     // [B << D] per-bucket Eytzinger tables of unit maxima images
    const uint32_t* gnode;   // two-level: one 32-B node of leaf-maxima images per unit
    const uint64_t* par;     // [2B] per-bucket image base, shift
    const uint32_t* mx;      // [B] global images of the bucket maxima
    const uint16_t* dir;     // [kBkBins + 1] radix directory over mx
    uint64_t gbase;          // global image: bk_img(x, gbase, gsh)
    uint32_t gsh;
    uint32_t Gp;             // CTAs of hist / part / unpart (tile t on CTA t % Gp)
    uint32_t Gs;             // CTAs of the search (one per SM)
    uint32_t CH;             // queries per search item
    uint32_t stream_hint;
    // workspace
    uint32_t* cnt;           // [G * B] per-CTA bucket counts -> exclusive prefix within the bucket
    uint32_t* tot;           // [B] bucket sizes
    K* rq;                   // [m] queries, bucket-major
    void* rp;                // [m] their results, same positions
    uint32_t* bp;            // [m] tile t's sorted position s: bucket | original slot << 16
    uint16_t* bkid;          // [m] bucket of query j (k_bk_hist -> k_bk_part)
    uint32_t* trun;          // [ntiles * B] (global position of run b) - (its sorted start), mod 2^32
    uint32_t* item_ctr;      // search items handed out (zeroed before the search)
    BucketPeer pr;           // fused peer return (pr.m_dev != NULL), params.h
};

// the batch size: m, or for the peer window (PM) the received count (capped
// at m).  A compile-time choice: a run-time one keeps m in registers for the
// whole kernel (measured: an 8-B spill in k_bk_part, +6 % on that pass)
template <bool PM, class K>
__device__ __forceinline__ uint64_t bk_m(const BkParams<K>& p) {
    if constexpr (!PM) {
        return p.m;
    } else {
        const uint64_t c = *(volatile const unsigned long long*)p.pr.m_dev;
        return c < p.m ? c : p.m;
    }
}

// bucket of x: #(bucket maxima < x).  The radix directory packs, per bin of
// the 32-bit global image, the candidate bucket range [lo, hi] (lo | hi << 16):
// #(maxima images < x's image) lies in it.  With more bins than buckets a bin
// holds at most one maximum almost always, so one predicated compare settles
// it; a bin with more maxima continues by bisection, and maxima whose image
// ties x's are compared exactly (galloping over the real maxima a[(j+1) NB - 1]).
template <class K>
__device__ __forceinline__ uint32_t bk_bucket_w(const BkParams<K>& p, const uint32_t* MS, uint32_t w, uint32_t fx, K x) {
    uint32_t l = w & 0xFFFFu, h = w >> 16;
    bool more = false, tie = false;
    if (l < h) {
        const uint32_t v = MS[l];
        const bool lt = v < fx;
        tie = v == fx;
        l += lt ? 1u : 0u;
        more = lt && l < h;   // a second maximum in the bin, and x above the first
    }
    if (__builtin_expect(more || tie, 0)) {
        // rare: more maxima in the bin, or an image tie
        while (l < h) {
            const uint32_t mid = (l + h) >> 1;
            if (MS[mid] < fx) l = mid + 1;
            else h = mid;
        }
        const uint32_t nm = p.B - 1;
        auto mxv = [&](uint32_t j) -> K { return ldg(p.a + ((uint64_t)j + 1) * p.NB - 1); };
        if (l < nm && MS[l] == fx && mxv(l) < x) {
            // step over the maxima that share x's image and are still < x: gallop, then bisect
            uint32_t lo = l + 1, step = 1, hi;
            for (;;) {
                hi = lo - 1 + step;
                if (hi >= nm) { hi = nm; break; }
                if (mxv(hi) >= x) break;
                lo = hi + 1;
                step <<= 1;
            }
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (mxv(mid) < x) lo = mid + 1;
                else hi = mid;
            }
            l = lo;
        }
    }
    return l;
}

// The common case of bk_bucket without branches: the bin's first candidate
// maximum decides unless the bin holds another maximum below x or an image
// ties x's; *rare is set for those, which the caller re-resolves with bk_bucket.
// D2[bin] = (lo | hi << 16, MS[lo]): the bin's candidate range and its first
// maximum in one 8-B shared load (one random shared access per query, not two)
template <class K>
__device__ __forceinline__ uint32_t bk_bucket_fast(const BkParams<K>& p, const uint2* D2, K x, uint32_t& fx,
                                                   uint32_t& w, bool& rare) {
    fx = bk_img((uint64_t)x, p.gbase, p.gsh);
    const uint2 d = D2[fx >> (32 - kBkBinsLog2)];
    w = d.x;
    const uint32_t l = w & 0xFFFFu, h = w >> 16;
    const uint32_t v = d.y;   // MS[l]: l <= B - 1 is always a maximum
    const bool has = l < h;
    const bool lt = has && v < fx;
    rare = (lt && l + 1 < h) || (has && v == fx);
    return l + (lt ? 1u : 0u);
}

// stage the bucket maxima images and the packed directory (plain loads; once per CTA)
template <class K>
__device__ __forceinline__ void bk_stage_dir2(const BkParams<K>& p, uint32_t* MS, uint2* D2) {
    for (uint32_t i = threadIdx.x; i < p.B; i += blockDim.x) MS[i] = p.mx[i];
    for (uint32_t i = threadIdx.x; i < kBkBins; i += blockDim.x) {
        const uint32_t lo = p.dir[i];
        D2[i] = make_uint2(lo | ((uint32_t)p.dir[i + 1] << 16), ldg(p.mx + lo));
    }
}

// block-wide exclusive scan of v[0..N) in place (blockDim.x = 1024); returns the total
__device__ __forceinline__ uint32_t bk_exscan(uint32_t* v, uint32_t N, uint32_t* tmp) {
    const uint32_t per = (N + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per;
    uint32_t s = 0;
    for (uint32_t i = 0; i < per; ++i)
        if (b0 + i < N) s += v[b0 + i];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
    }
    if (lane == 31) tmp[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = lane < (blockDim.x >> 5) ? tmp[lane] : 0u;
        uint32_t wi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= (uint32_t)o) wi += y;
        }
        tmp[lane] = wi - x;
        if (lane == 31) tmp[32] = wi;
    }
    __syncthreads();
    uint32_t run = tmp[w] + inc - s;
    for (uint32_t i = 0; i < per; ++i) {
        if (b0 + i < N) {
            const uint32_t c = v[b0 + i];
            v[b0 + i] = run;
            run += c;
        }
    }
    const uint32_t total = tmp[32];
    __syncthreads();
    return total;
}

// two consecutive keys with one vector load (16 B for u64, 8 B for u32), streaming
template <class K>
__device__ __forceinline__ void ld_pair(const K* p, uint64_t pol, K& x0, K& x1) {
    if constexpr (sizeof(K) == 8) {
        uint64_t a, b;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                     : "=l"(a), "=l"(b) : "l"(p), "l"(pol));
        x0 = a; x1 = b;
    } else {
        uint32_t a, b;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                     : "=r"(a), "=r"(b) : "l"(p), "l"(pol));
        x0 = a; x1 = b;
    }
}

// ---- pass 1: per-CTA histograms (same tile -> CTA map as k_bk_part); the next
// tile's queries are in flight while this tile is bucketed.  Each thread takes
// pairs of neighbouring queries (one vector load, one 4-B store of the two
// bucket ids): the pass is issue-bound, not bandwidth-bound.
template <class K, bool PM>
__global__ void __launch_bounds__(kBkPThreads, kBkPCtas)
k_bk_hist(const BkParams<K> p) {
    constexpr uint32_t T = kBkTile, E2 = T / kBkPThreads / 2;   // pairs per thread per tile
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t B4 = (p.B + 3u) & ~3u;
    uint32_t* MS = sm;
    uint32_t* hist = MS + B4;
    uint2* D2 = reinterpret_cast<uint2*>(hist + B4);          // [kBkBins] (lo | hi << 16, MS[lo])
    bk_stage_dir2(p, MS, D2);
    for (uint32_t b = threadIdx.x; b < p.B; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const uint64_t pol = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t m = bk_m<PM>(p);
    const uint64_t ntiles = (m + T - 1) / T;
    // vector loads need the batch 2-key aligned (bs_lookup only requires key alignment)
    const bool pairs_ok = ((uintptr_t)p.q & (2 * sizeof(K) - 1)) == 0;
    auto load_tile = [&](uint64_t t, K* xs) {
        const uint64_t b0 = t * T;
        const bool full = pairs_ok && t < ntiles && b0 + T <= m;
#pragma unroll
        for (uint32_t e = 0; e < E2; ++e) {
            const uint64_t j = b0 + 2 * (e * kBkPThreads + threadIdx.x);
            if (full) {
                ld_pair<K>(p.q + j, pol, xs[2 * e], xs[2 * e + 1]);
            } else {
                xs[2 * e] = (t < ntiles && j < m) ? load_stream(p.q + j, true, pol) : (K)0;
                xs[2 * e + 1] = (t < ntiles && j + 1 < m) ? load_stream(p.q + j + 1, true, pol) : (K)0;
            }
        }
    };
    constexpr bool PF = E2 <= 4;   // the next tile in flight when the registers allow it
    K xn[PF ? 2 * E2 : 1];
    if constexpr (PF) load_tile(blockIdx.x, xn);
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t b0 = t * T;
        const uint32_t cntq = (uint32_t)((m - b0) < T ? (m - b0) : T);
        K x[2 * E2];
        if constexpr (PF) {
#pragma unroll
            for (uint32_t e = 0; e < 2 * E2; ++e) x[e] = xn[e];
            load_tile(t + gridDim.x, xn);
        } else {
            load_tile(t, x);
        }
        if (cntq == T) {
            // full tile: each pair's buckets branch-free, a pair with a rare query
            // (a second maximum in the bin, an image tie) re-resolved exactly —
            // the pass is issue-bound, and branches per query cost reconvergences
#pragma unroll
            for (uint32_t e = 0; e < E2; ++e) {
                const uint32_t j = 2 * (e * kBkPThreads + threadIdx.x);
                bool r0, r1;
                uint32_t f0, f1, w0, w1;
                uint32_t b0v = bk_bucket_fast(p, D2, x[2 * e], f0, w0, r0);
                uint32_t b1v = bk_bucket_fast(p, D2, x[2 * e + 1], f1, w1, r1);
                if (__builtin_expect(r0 || r1, 0)) {
                    b0v = bk_bucket_w(p, MS, w0, f0, x[2 * e]);
                    b1v = bk_bucket_w(p, MS, w1, f1, x[2 * e + 1]);
                }
                atomicAdd(&hist[b0v], 1u);
                atomicAdd(&hist[b1v], 1u);
                // the partition pass reads the bucket ids back
                __stcs(reinterpret_cast<uint32_t*>(p.bkid + b0 + j), b0v | (b1v << 16));
            }
            continue;
        }
#pragma unroll
        for (uint32_t e = 0; e < E2; ++e) {
            const uint32_t j = 2 * (e * kBkPThreads + threadIdx.x);
            uint32_t b01 = 0;
#pragma unroll
            for (uint32_t h = 0; h < 2; ++h) {
                if (j + h < cntq) {
                    const uint32_t fx = bk_img((uint64_t)x[2 * e + h], p.gbase, p.gsh);
                    const uint32_t b = bk_bucket_w(p, MS, D2[fx >> (32 - kBkBinsLog2)].x, fx, x[2 * e + h]);
                    atomicAdd(&hist[b], 1u);
                    b01 |= b << (16 * h);
                }
            }
            // the partition pass reads the bucket ids back
            if (j + 1 < cntq) __stcs(reinterpret_cast<uint32_t*>(p.bkid + b0 + j), b01);
            else if (j < cntq) __stcs(p.bkid + b0 + j, (uint16_t)b01);
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < p.B; b += blockDim.x) p.cnt[(uint64_t)blockIdx.x * p.B + b] = hist[b];
}

// ---- pass 2: per bucket, the exclusive prefix of the G CTA counts (32 buckets per CTA)
__global__ void __launch_bounds__(1024)
k_bk_scan(uint32_t* __restrict__ cnt, uint32_t* __restrict__ tot, uint32_t G, uint32_t B) {
    __shared__ uint32_t part[32][33];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t b = blockIdx.x * 32 + lane;
    const uint32_t c0 = G * w / 32, c1 = G * (w + 1) / 32;
    uint32_t s = 0;
    if (b < B)
        for (uint32_t c = c0; c < c1; ++c) s += cnt[(uint64_t)c * B + b];
    part[w][lane] = s;
    __syncthreads();
    if (w == 0) {
        uint32_t run = 0;
        for (uint32_t i = 0; i < 32; ++i) {
            const uint32_t v = part[i][lane];
            part[i][lane] = run;
            run += v;
        }
        if (b < B) tot[b] = run;
    }
    __syncthreads();
    if (b < B) {
        uint32_t run = part[w][lane];
        for (uint32_t c = c0; c < c1; ++c) {
            const uint64_t o = (uint64_t)c * B + b;
            const uint32_t v = cnt[o];
            cnt[o] = run;
            run += v;
        }
    }
}

// a query and its (bucket, slot) word side by side in the sorted tile: one
// 16-B (u64) / 8-B (u32) shared store and load per query instead of two each
template <class K> struct BkPair;
template <> struct alignas(16) BkPair<uint64_t> { uint64_t k; uint32_t bp, pad; };
template <> struct alignas(8) BkPair<uint32_t> { uint32_t k; uint32_t bp; };

template <class K>
__device__ __forceinline__ void st_pair(BkPair<K>* d, K k, uint32_t bp) {
    if constexpr (sizeof(K) == 8) *reinterpret_cast<uint4*>(d) = make_uint4((uint32_t)k, (uint32_t)(k >> 32), bp, 0u);
    else *reinterpret_cast<uint2*>(d) = make_uint2((uint32_t)k, bp);
}
template <class K>
__device__ __forceinline__ void ld_pair_smem(const BkPair<K>* s, K& k, uint32_t& bp) {
    if constexpr (sizeof(K) == 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(s);
        k = ((uint64_t)v.y << 32) | v.x;
        bp = v.z;
    } else {
        const uint2 v = *reinterpret_cast<const uint2*>(s);
        k = v.x;
        bp = v.y;
    }
}

// ---- pass 3: partition (tile t on CTA t % G, as in k_bk_hist)
//
// Thread i owns buckets [i BPT, (i+1) BPT) (BPT = kBkFineMax / threads = 1): their
// tile counts, run starts and global cursors live in its registers, so a tile
// costs four barriers (ranks / warp totals / run starts / sorted tile) and no
// loops over the buckets; the next tile's queries and bucket ids are in flight
// while this tile is sorted and stored.
template <class K, bool PM>
__global__ void __launch_bounds__(kBkPThreads, kBkPCtas)
k_bk_part(const BkParams<K> p) {
    constexpr uint32_t T = kBkTile, E = T / kBkPThreads, BPT = kBkFineMax / kBkPThreads;
    constexpr uint32_t NW = kBkPThreads / 32;
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t B = p.B;
    BkPair<K>* st = reinterpret_cast<BkPair<K>*>(sm);         // [T] query + (bucket | original slot << 16), bucket order
    uint32_t* hist = reinterpret_cast<uint32_t*>(st + T);     // [kBkFineMax] tile counts (ranks by atomics)
    uint32_t* loff = hist + kBkFineMax;                       // [kBkFineMax] tile run starts (sorted order)
    uint32_t* rbase = loff + kBkFineMax;                      // [kBkFineMax] global position of run b minus its sorted start
    uint32_t* wsum = rbase + kBkFineMax;                      // [NW] warp totals
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t b_lo = threadIdx.x * BPT;
    // this CTA's next global position per owned bucket: the bucket's start (an
    // exclusive scan of the bucket sizes) + this CTA's prefix within the bucket
    uint32_t cur[BPT];
    {
        uint32_t own = 0;
#pragma unroll
        for (uint32_t k = 0; k < BPT; ++k) {
            cur[k] = b_lo + k < B ? p.tot[b_lo + k] : 0u;
            own += cur[k];
            hist[b_lo + k] = 0;
        }
        uint32_t inc = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t run = inc - own;
        for (uint32_t w = 0; w < warp; ++w) run += wsum[w];
#pragma unroll
        for (uint32_t k = 0; k < BPT; ++k) {
            const uint32_t c = cur[k];
            cur[k] = run + (b_lo + k < B ? p.cnt[(uint64_t)blockIdx.x * B + b_lo + k] : 0u);
            run += c;
        }
    }
    const uint64_t pol = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_run = policy_evict_normal();
    // PM: the received count is re-read from shared memory at each use — held
    // in registers across the kernel it costs an 8-B spill (64 registers)
    __shared__ unsigned long long s_m;
    if constexpr (PM) {
        if (threadIdx.x == 0) s_m = bk_m<true>(p);
        __syncthreads();
    }
    auto M = [&]() -> uint64_t {
        if constexpr (PM) return *(volatile unsigned long long*)&s_m;
        else return p.m;
    };
    const uint64_t ntiles = (M() + T - 1) / T;
    constexpr bool PF = E <= 8;   // the next tile in flight when the registers allow it
    K xn[PF ? E : 1];
    uint32_t bn[PF ? E : 1];
    auto load_tile = [&](uint64_t t, K* xs, uint32_t* bs) {
        const uint64_t b0 = t * T;
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            const uint64_t j = b0 + e * kBkPThreads + threadIdx.x;
            const bool ok = t < ntiles && j < M();
            xs[e] = ok ? load_stream(p.q + j, true, pol) : (K)0;
            bs[e] = ok ? (uint32_t)__ldcs(p.bkid + j) : 0xFFFFu;   // from k_bk_hist
        }
    };
    if constexpr (PF) load_tile(blockIdx.x, xn, bn);
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t b0 = t * T;
        const uint32_t cntq = (uint32_t)((M() - b0) < T ? (M() - b0) : T);
        K x[E];
        uint32_t br[E];   // bucket | rank in the tile's run << 16
        if constexpr (PF) {
#pragma unroll
            for (uint32_t e = 0; e < E; ++e) { x[e] = xn[e]; br[e] = bn[e]; }
            load_tile(t + gridDim.x, xn, bn);
        } else {
            load_tile(t, x, br);
        }
        __syncthreads();   // (1) hist is zero and the previous tile's readout is done
#pragma unroll
        for (uint32_t e = 0; e < E; ++e)
            if (br[e] != 0xFFFFu) br[e] |= atomicAdd(&hist[br[e]], 1u) << 16;
        __syncthreads();   // (2) the tile's counts are final
        uint32_t c[BPT], own = 0;
#pragma unroll
        for (uint32_t k = 0; k < BPT; ++k) {
            c[k] = hist[b_lo + k];
            hist[b_lo + k] = 0;
            own += c[k];
        }
        uint32_t inc = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();   // (3) warp totals
        // this warp's offset: exclusive scan of the warp totals across the lanes
        uint32_t ws = lane < NW ? wsum[lane] : 0u, wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= (uint32_t)o) wi += y;
        }
        uint32_t run = inc - own + __shfl_sync(0xFFFFFFFFu, wi - ws, warp);
#pragma unroll
        for (uint32_t k = 0; k < BPT; ++k) {
            // the run of bucket b starts at cur[b] in the bucket-major array: P3 finds a
            // sorted position s of bucket b there at (cur[b] - loff[b]) + s
            const uint32_t b = b_lo + k;
            const uint32_t rb = cur[k] - run;
            loff[b] = run;
            rbase[b] = rb;
            if (b < B) p.trun[t * B + b] = rb;
            cur[k] += c[k];
            run += c[k];
        }
        __syncthreads();   // (4) run starts
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            if (br[e] == 0xFFFFu) continue;
            const uint32_t b = br[e] & 0xFFFFu;
            const uint32_t sidx = loff[b] + (br[e] >> 16);
            st_pair<K>(st + sidx, x[e], b | ((e * kBkPThreads + threadIdx.x) << 16));
        }
        __syncthreads();   // (5) the sorted tile
        // each run to its place in its bucket's region (consecutive within a run;
        // evict_normal: the run's partial lines are completed by this CTA's next
        // tile and must stay in L2 until then), and the tile's (bucket, slot) list
        for (uint32_t sidx = threadIdx.x; sidx < cntq; sidx += blockDim.x) {
            K k;
            uint32_t w;
            ld_pair_smem<K>(st + sidx, k, w);
            store_stream(p.rq + (uint32_t)(rbase[w & 0xFFFFu] + sidx), k, true, pol_run);
            store_stream(p.bp + b0 + sidx, w, true, pol);
        }
    }
}

// ---- pass 4: the per-bucket search
//
// One lookup: x's image under the bucket's parameters descends D levels of the
// staged table (one 4-B shared load per level on the address recurrence
// a' = 2a - sb + 4 [T[k] < q]), which gives u = #(unit maxima images < q's) <=
// the exact unit.  Fine buckets (G = 1): a unit is one 32-B leaf.  Two-level
// buckets (G = 8, arrays above 2^27 u64 keys): a unit is a group of 8 leaves of
// 64 B, and one 32-B global node of the 8 leaf maxima images (L2-hot) picks the
// leaf: the next three levels of the same tree, kept in L2.  The leaf gives lb;
// a leaf whose keys are all < q (possible only when a maximum's image ties q's)
// continues by galloping over the real leaf maxima.
template <class K, int OB, int LV>
__device__ __forceinline__ void bk_finish(const K* __restrict__ ab, uint64_t klo, uint64_t len, uint32_t Mb,
                                          uint64_t n, K x, uint32_t c, const uint64_t* lv, void* rp, uint32_t ir,
                                          uint64_t pol_leaf, uint64_t pol_stream) {
    using O = typename std::conditional<OB == 8, uint64_t, uint32_t>::type;
    constexpr uint32_t LK = 8u * LV / sizeof(K);
    uint64_t lb;
    bool hit = false;
    if (c >= Mb) {
        lb = n;   // past every key of the (last) bucket
    } else {
        uint32_t nlt = 0;
        bool eq = false;
#pragma unroll
        for (uint32_t u = 0; u < LK; ++u) {
            const K v = bk_key<K>(lv, (int)u);
            nlt += v < x ? 1u : 0u;
            eq |= v == x;
        }
        if (nlt == LK && c + 1 < Mb) {
            // leaf maxima whose image ties q's may still be < q: gallop over the
            // real maxima to the first >= q, then rescan that leaf
            auto mxv = [&](uint32_t j) -> K {
                const uint64_t e = ((uint64_t)j + 1) * LK;
                return ldg(ab + (e < len ? e : len) - 1);
            };
            uint32_t l = c + 1, step = 1, h;
            for (;;) {
                h = l - 1 + step;
                if (h >= Mb) { h = Mb; break; }
                if (mxv(h) >= x) break;
                l = h + 1;
                step <<= 1;
            }
            while (l < h) {
                const uint32_t mid = (l + h) >> 1;
                if (mxv(mid) < x) l = mid + 1;
                else h = mid;
            }
            c = l;
            nlt = 0;
            eq = false;
            if (l < Mb) {
                for (uint32_t u = 0; u < LK; ++u) {
                    const K v = ldg(ab + (uint64_t)l * LK + u);
                    nlt += v < x ? 1u : 0u;
                    eq |= v == x;
                }
            }
        }
        lb = klo + (uint64_t)c * LK + nlt;
        if (lb > n) lb = n;
        hit = eq && lb < n;
    }
    constexpr uint64_t MISS = 1ull << (8 * OB - 1);
    store_stream((O*)rp + ir, (O)(hit ? lb : (lb | MISS)), true, pol_stream);
}

// Items of CH queries in bucket order, handed out by a global counter (the CTAs
// work on a window of neighbouring buckets, whose slices of the array stay in
// L2); the bucket's table is staged once per item that changes bucket.  R
// lookups per thread descend together (their shared-memory latencies overlap).
// Measured alternative: a software pipeline (leaves of batch k in flight while
// batch k+1 descends) ran 3 % slower — the kernel is bound by the L1 data pipe
// (shared-memory bank conflicts of the random probes + one leaf wavefront per
// lookup), not by latency.
// threads of the search: 768 for 16-leaf units (80 registers: the node and the
// leaf of two lookups in flight), else 1024
constexpr uint32_t bk_search_threads(int G) { return G == 16 ? 768u : kBkThreads; }

template <class K, int OB, int D, int G, int LV>
__global__ void __launch_bounds__(bk_search_threads(G), 1)
k_bk_search(const BkParams<K> p) {
    // LV: leaf size in u64 words (4: 32 B, 8: 64 B)
    constexpr uint32_t LK = 8u * LV / sizeof(K);            // keys per leaf
    constexpr uint32_t R = (G == 1 && LV == 4) ? 4 : 2;    // lookups in flight per thread
    constexpr uint32_t TS = bk_search_threads(G);
    constexpr uint32_t S = 1u << D;
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t B = p.B;
    uint32_t* Tab = sm;                                     // [2^D]
    uint32_t* bst = Tab + S;                                // [B + 1] bucket starts
    uint32_t* ipre = bst + ((B + 4u) & ~3u);                // [B + 1] first item of each bucket
    uint32_t* tmp = ipre + ((B + 4u) & ~3u);                // [64]
    uint64_t* bar = reinterpret_cast<uint64_t*>(tmp + 64);
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) {
        const uint32_t t = p.tot[b];
        bst[b] = t;
        ipre[b] = (t + p.CH - 1) / p.CH;
    }
    __syncthreads();
    const uint32_t mtot = bk_exscan(bst, B, tmp);
    const uint32_t I = bk_exscan(ipre, B, tmp);
    if (threadIdx.x == 0) { bst[B] = mtot; ipre[B] = I; }
    __syncthreads();
    const uint64_t pol_stream = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_leaf = policy_evict_normal();
    const uint32_t sb = smem_u32(Tab);
    const uint32_t step_lt = 4u - sb, step_ge = 0u - sb;
    uint32_t staged = 0xFFFFFFFFu;
    // items in bucket order from a global counter: every CTA stays within one
    // item of the front, so the CTAs work on a window of neighbouring buckets
    // for the whole batch (a static item stride lets them drift apart)
    uint32_t* s_it = tmp + 48;
    for (;;) {
        __syncthreads();   // s_it free; every lookup of the previous item is issued
        if (threadIdx.x == 0) *s_it = atomicAdd(p.item_ctr, 1u);
        __syncthreads();
        const uint32_t it = *s_it;
        if (it >= I) break;
        // bucket of item it: the last b with ipre[b] <= it (it has items, so ipre[b+1] > it)
        uint32_t lo = 0, hi = B;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ipre[mid] <= it) lo = mid;
            else hi = mid;
        }
        const uint32_t b = lo;
        const uint32_t i0 = bst[b] + (it - ipre[b]) * p.CH;
        const uint32_t i1 = min(i0 + p.CH, bst[b + 1]);
        if (b != staged) {
            __syncthreads();   // every lookup of the previous item is done with Tab
            stage_to_smem(Tab, p.tab + ((uint64_t)b << D), 4u << D, bar);
            staged = b;
        }
        const uint64_t base = p.par[2 * b];
        const uint32_t sh = (uint32_t)p.par[2 * b + 1];
        const uint64_t klo = (uint64_t)b * p.NB;
        const uint64_t len = (p.n - klo) < p.NB ? (p.n - klo) : p.NB;
        const uint32_t Mb = (uint32_t)((len + LK - 1) / LK);   // leaves holding keys
        const K* ab = p.a + klo;
        // G = 8: u32 leaf-maxima images, 8 per unit; G = 16: u16 images relative to the unit
        const uint32_t* gn = p.gnode + ((uint64_t)b << D) * (G == 16 ? G / 2 : G);
        for (uint32_t i = i0 + threadIdx.x; i < i1; i += TS * R) {
            K x[R];
            uint32_t ad[R], fq[R];
            uint32_t flo[G == 16 ? R : 1], fhi[G == 16 ? R : 1];   // the unit's image range (G = 16)
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) {
                const uint32_t ir = i + r * TS;
                x[r] = ir < i1 ? load_stream(p.rq + ir, true, pol_stream) : (K)base;
                fq[r] = bk_img((uint64_t)x[r], base, sh);
                ad[r] = sb + 4u;
                if constexpr (G == 16) { flo[r] = 0u; fhi[r] = 0xFFFFFFFFu; }
            }
#pragma unroll
            for (uint32_t d = 0; d < (uint32_t)D; ++d) {
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    const uint32_t h = lds_u32(ad[r]);
                    const bool lt = h < fq[r];
                    ad[r] = 2u * ad[r] + (lt ? step_lt : step_ge);
                    if constexpr (G == 16) {
                        flo[r] = lt ? h : flo[r];
                        fhi[r] = lt ? fhi[r] : h;
                    }
                }
            }
            uint32_t c[R];
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) c[r] = ((ad[r] - sb) >> 2) - S;   // unit
            if constexpr (G == 16) {
                // the unit's node of 16 leaf-maxima images relative to [flo, fhi] (32 B, one
                // sector): leaf = 16 u + #(< q's relative image)
                uint64_t nd[R][4];
#pragma unroll
                for (uint32_t r = 0; r < R; ++r)
                    if (c[r] * G < Mb) ld_sector(gn + (uint64_t)c[r] * (G / 2), pol_leaf, nd[r]);
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    const uint32_t q16 = (fq[r] - flo[r]) >> bk_sub_shift(flo[r], fhi[r]);   // fq > flo
                    uint32_t j = 0;
#pragma unroll
                    for (uint32_t k = 0; k < 16; ++k) {
                        const uint32_t im = (uint32_t)(nd[r][k >> 2] >> (16 * (k & 3))) & 0xFFFFu;
                        j += im < q16 ? 1u : 0u;
                    }
                    c[r] = c[r] * G < Mb ? c[r] * G + j : Mb;
                }
            } else if constexpr (G > 1) {
                // the unit's node of G leaf maxima images (32 B, one sector): leaf = G u + #(< q)
                uint64_t nd[R][4];
#pragma unroll
                for (uint32_t r = 0; r < R; ++r)
                    if (c[r] * G < Mb) ld_sector(gn + (uint64_t)c[r] * G, pol_leaf, nd[r]);
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    uint32_t j = 0;
#pragma unroll
                    for (uint32_t k = 0; k < 8; ++k) {
                        const uint32_t im = (uint32_t)(nd[r][k >> 1] >> (32 * (k & 1)));
                        j += im < fq[r] ? 1u : 0u;
                    }
                    c[r] = c[r] * G < Mb ? c[r] * G + j : Mb;
                }
            }
            uint64_t lv[R][LV];
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) {
                if (c[r] < Mb) {
#pragma unroll
                    for (uint32_t h = 0; h < LV; h += 4) ld_sector(ab + (uint64_t)c[r] * LK + h * (8 / sizeof(K)), pol_leaf, &lv[r][h]);
                }
            }
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) {
                const uint32_t ir = i + r * TS;
                if (ir < i1) bk_finish<K, OB, LV>(ab, klo, len, Mb, p.n, x[r], c[r], lv[r], p.rp, ir, pol_leaf, pol_stream);
            }
        }
    }
}

// ---- pass 5: back to query order (any grid: the run bases are stored per tile)
template <class K, int OB, bool PM>
__global__ void __launch_bounds__(kBkPThreads, kBkUCtas)
k_bk_unpart(const BkParams<K> p) {
    using O = typename std::conditional<OB == 8, uint64_t, uint32_t>::type;
    constexpr uint32_t T = kBkTile, E = T / kBkPThreads;
    extern __shared__ __align__(16) uint32_t sm[];
    O* so = reinterpret_cast<O*>(sm);                         // [T] results, query order
    uint32_t* rb = reinterpret_cast<uint32_t*>(so + T);       // [B]
    const uint32_t B = p.B;
    const uint64_t pol = p.stream_hint ? policy_evict_first() : policy_evict_normal();
    const uint64_t m = bk_m<PM>(p);
    const uint64_t ntiles = (m + T - 1) / T;
    const uint64_t pol_run = policy_evict_normal();   // runs share lines with the neighbouring tiles' runs
    const O* rp = (const O*)p.rp;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t b0 = t * T;
        const uint32_t cntq = (uint32_t)((m - b0) < T ? (m - b0) : T);
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) rb[b] = p.trun[t * B + b];
        uint32_t bp[E];   // bucket | slot << 16
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            const uint32_t s = e * kBkPThreads + threadIdx.x;
            bp[e] = s < cntq ? load_stream(p.bp + b0 + s, true, pol) : 0u;
        }
        __syncthreads();   // rb is in place; the previous tile's stores have read `so`
        // gathers in two halves of E/2 loads in flight (32 registers: two CTAs per SM)
#pragma unroll
        for (uint32_t h = 0; h < E; h += E / 2) {
            O v[E / 2];
#pragma unroll
            for (uint32_t e = 0; e < E / 2; ++e) {
                const uint32_t s = (h + e) * kBkPThreads + threadIdx.x;
                if (s < cntq) v[e] = load_stream(rp + (uint32_t)(rb[bp[h + e] & 0xFFFFu] + s), true, pol_run);
            }
#pragma unroll
            for (uint32_t e = 0; e < E / 2; ++e) {
                const uint32_t s = (h + e) * kBkPThreads + threadIdx.x;
                if (s < cntq) so[bp[h + e] >> 16] = v[e];
            }
        }
        __syncthreads();
        if constexpr (PM && OB == 8) {
            {
                // fused peer return: window slot b0 + j's result, made global (+ the
                // shard's base), straight into its source rank's return window
                constexpr uint64_t MISS = 1ull << 63;
                const uint32_t sh = p.pr.shift;
                const uint64_t msk = (1ull << sh) - 1ull;
                for (uint32_t j = threadIdx.x; j < cntq; j += blockDim.x) {
                    const uint32_t tg = __ldcg(p.pr.tag + b0 + j);
                    const uint64_t v = (uint64_t)so[j];
                    const uint64_t g = (v & ~MISS) + p.pr.base;
                    p.pr.ret[(uint64_t)tg >> sh][tg & msk] = (v & MISS) ? (g | MISS) : g;
                }
                continue;
            }
        }
        O* out = (O*)p.out + b0;
        if (cntq == T && OB == 8 && ((uintptr_t)p.out & 15) == 0) {
            // 16-B stores: two results per thread per step
            for (uint32_t j = threadIdx.x * 2; j < T; j += blockDim.x * 2) {
                const uint2 lo = *reinterpret_cast<const uint2*>(so + j);
                const uint2 hi = *reinterpret_cast<const uint2*>(so + j + 1);
                asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
                             :: "l"(out + j), "r"(lo.x), "r"(lo.y), "r"(hi.x), "r"(hi.y), "l"(pol) : "memory");
            }
        } else {
            for (uint32_t j = threadIdx.x; j < cntq; j += blockDim.x) store_stream(out + j, so[j], true, pol);
        }
    }
    if constexpr (PM && OB == 8) {
        if (peer_last_cta(p.pr.done)) {
            // every CTA has read the cursor and stored its results: re-arm the
            // window, then tell every rank its results have landed
            *p.pr.cursor = 0;
            __threadfence_system();
            for (uint32_t r = 0; r < p.pr.P; ++r) red_release_sys_add_u64(p.pr.sig[r], 1ull);
        }
    }
}

// ------------------------------------------------------------------ host

struct BkLayout {
    uint64_t G, Gs, B, ntiles;
    uint64_t o_cnt, o_tot, o_rq, o_rp, o_bp, o_bkid, o_trun, o_ctr, total;
};

static bool bk_layout(uint64_t B, uint64_t m, int kb, int ob, uint32_t sm_count, BkLayout* L) {
    if (B == 0 || B > kBkMaxBuckets || m >= (1ull << 32)) return false;
    L->G = (uint64_t)kBkPCtas * sm_count;   // CTAs of hist / part (unpart runs twice as many)
    L->Gs = sm_count;
    L->B = B;
    L->ntiles = (m + kBkTile - 1) / kBkTile;
    const uint64_t mm = m ? m : 1;
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) { const uint64_t r = o; o += (bytes + 255) & ~255ull; return r; };
    L->o_cnt = take(4 * L->G * B);
    L->o_tot = take(4 * B);
    L->o_rq = take((uint64_t)kb * mm);
    L->o_rp = take((uint64_t)ob * mm);
    L->o_bp = take(4 * mm);
    L->o_bkid = take(2 * mm);
    L->o_trun = take(4 * L->ntiles * B);
    L->o_ctr = take(4);
    L->total = o;
    return true;
}

bool bucket_workspace_bytes(uint64_t B, uint64_t m, int kb, int ob, uint32_t sm_count, uint64_t* bytes) {
    BkLayout L;
    if (!bk_layout(B, m, kb, ob, sm_count, &L)) return false;
    *bytes = L.total;
    return true;
}

static cudaError_t bk_launch(const void* kern, uint32_t threads, uint32_t smem, uint32_t blocks, const void* params,
                             cudaStream_t s) {
    bool uns = false;
    uint64_t g = 0;
    Grid grid{0u, 1u, blocks};
    cudaError_t e = plan_grid(kern, threads, smem, grid, blocks, carveout_for(smem, threads), &g, &uns);
    if (e != cudaSuccess) return e;
    if (uns) return cudaErrorInvalidConfiguration;
    void* args[] = {const_cast<void*>(params)};
    e = cudaLaunchKernel(kern, dim3(blocks), dim3(threads), args, smem, s);
    count_launch();
    return e;
}

template <class K, int OB>
static cudaError_t go_bucket(BkParams<K> p, const BkLayout& L, char* ws, cudaStream_t s, int phase, BucketRun* run) {
    p.Gp = (uint32_t)L.G;
    p.Gs = (uint32_t)L.Gs;
    p.cnt = (uint32_t*)(ws + L.o_cnt);
    p.tot = (uint32_t*)(ws + L.o_tot);
    p.rq = (K*)(ws + L.o_rq);
    p.rp = ws + L.o_rp;
    p.bp = (uint32_t*)(ws + L.o_bp);
    p.bkid = (uint16_t*)(ws + L.o_bkid);
    p.trun = (uint32_t*)(ws + L.o_trun);
    p.item_ctr = (uint32_t*)(ws + L.o_ctr);
    if (run) { run->rq = p.rq; run->rp = p.rp; }
    const bool pm = p.pr.m_dev != nullptr;   // the peer window (size on the device)
    const uint32_t B = p.B, B4 = (B + 3u) & ~3u;
    cudaError_t e;
    if (phase != 2) {
        {
            const uint32_t smem = 8u * B4 + 8u * kBkBins;
            e = bk_launch(pm ? (const void*)k_bk_hist<K, true> : (const void*)k_bk_hist<K, false>, kBkPThreads, smem, p.Gp, &p, s);
            if (e != cudaSuccess) return e;
        }
        k_bk_scan<<<(B + 31) / 32, 1024, 0, s>>>(p.cnt, p.tot, p.Gp, B);
        count_launch();
        {
            const uint32_t smem = kBkTile * (uint32_t)sizeof(BkPair<K>) + 4u * (3u * kBkFineMax + 32u);
            e = bk_launch(pm ? (const void*)k_bk_part<K, true> : (const void*)k_bk_part<K, false>, kBkPThreads, smem, p.Gp, &p, s);
            if (e != cudaSuccess) return e;
        }
    }
    if (phase == 0) {
        const uint32_t smem = (4u << p.D) + 8u * ((B + 4u) & ~3u) + 4u * 64u + 16u;
        const void* kern = nullptr;
        if (p.gnode && p.D == 15) kern = p.G == 16 ? (const void*)k_bk_search<K, OB, 15, 16, 4>
                                       : p.LB == 32 ? (const void*)k_bk_search<K, OB, 15, 8, 4>
                                                    : (const void*)k_bk_search<K, OB, 15, 8, 8>;
        else if (!p.gnode) kern = p.D == 15 ? (const void*)k_bk_search<K, OB, 15, 1, 4>
                                : p.D == 14 ? (const void*)k_bk_search<K, OB, 14, 1, 4> : nullptr;
        if (!kern) return cudaErrorInvalidValue;
        e = cudaMemsetAsync(p.item_ctr, 0, sizeof(uint32_t), s);
        if (e != cudaSuccess) return e;
        e = bk_launch(kern, bk_search_threads(p.gnode ? (int)p.G : 1), smem, p.Gs, &p, s);
        if (e != cudaSuccess) return e;
    }
    if (phase != 1) {
        const uint32_t smem = kBkTile * OB + 4u * B4;
        const void* ku = (const void*)k_bk_unpart<K, OB, false>;
        if constexpr (OB == 8) {
            if (pm) ku = (const void*)k_bk_unpart<K, 8, true>;   // the peer return (out_bytes 8 only)
        }
        e = bk_launch(ku, kBkPThreads, smem, kBkUCtas * p.Gs, &p, s);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

cudaError_t launch_bucket(int kb, int ob, const BucketIndex& bi, const void* a, uint64_t n, const void* q, uint64_t m,
                          void* out, uint32_t stream_hint, uint32_t chunk, void* ws, uint64_t ws_bytes,
                          uint32_t sm_count, cudaStream_t s, bool* uns, int phase, BucketRun* run,
                          const BucketPeer* peer) {
    BkLayout L;
    if (!bi.mx || (phase == 0 && !bi.tab) || !bk_layout(bi.B, m, kb, ob, sm_count, &L) || ws_bytes < L.total ||
        (peer && (phase != 0 || ob != 8 || !peer->m_dev))) {
        *uns = true;
        return cudaSuccess;
    }
    auto fill = [&](auto& p) {
        p.n = n; p.m = m; p.out = out; p.stream_hint = stream_hint;
        p.B = (uint32_t)bi.B; p.D = bi.D; p.NB = bi.NB; p.LB = bi.LB; p.G = bi.G;
        p.tab = bi.tab; p.par = bi.par; p.mx = bi.mx; p.dir = bi.dir; p.gnode = bi.gnode;
        p.gbase = bi.gbase; p.gsh = bi.gsh;
        if (peer) p.pr = *peer;
        const uint64_t mi = peer && peer->m_hint ? peer->m_hint : m;
        // search items: the CTAs' window of items spans ~37 MB of keys (config 3:
        // 37 fine buckets of 1 MB; config 4: ~2.3 two-level buckets of 16 MB),
        // at most kBkChunk (the config-3 optimum) and at least 16384 queries:
        // with fewer queries per bucket each leaf line is read about once per
        // batch whatever the window, and a smaller item only adds table stagings
        // (measured: 2^24 queries at config-3 keys 0.465 -> 0.449 ms, config 5
        // 9.75 -> 9.38 ms with the 16384 floor instead of 4096)
        uint64_t ch = chunk;
        if (!ch) {
            const uint64_t bucket_bytes = bi.NB * (uint64_t)kb;
            ch = (uint64_t)((double)mi * (37.0 * (1 << 20) / (double)bucket_bytes) / ((double)sm_count * (double)bi.B));
            ch = ch > kBkChunk ? kBkChunk : (ch < 16384 ? 16384 : ch);
        }
        p.CH = (uint32_t)ch;
    };
    if (kb == 8) {
        BkParams<uint64_t> p{};
        fill(p);
        p.a = (const uint64_t*)a; p.q = (const uint64_t*)q;
        return ob == 8 ? go_bucket<uint64_t, 8>(p, L, (char*)ws, s, phase, run)
                       : go_bucket<uint64_t, 4>(p, L, (char*)ws, s, phase, run);
    }
    BkParams<uint32_t> p{};
    fill(p);
    p.a = (const uint32_t*)a; p.q = (const uint32_t*)q;
    return ob == 8 ? go_bucket<uint32_t, 8>(p, L, (char*)ws, s, phase, run)
                   : go_bucket<uint32_t, 4>(p, L, (char*)ws, s, phase, run);
}

}  // namespace bs
