// build.cu — index construction kernels (bs_build; not on the lookup path).
//   * unsigned radix sort of a key copy (CUB DeviceRadixSort) when the caller's
//     keys are not declared sorted;
//   * sortedness check when they are;
//   * level-major pinned table (§4.2): T[base_d + k] = a[n-1-(2k+1)(s0>>d)];
//   * K-ary separator levels (§5): slot j of node m at level l (top-first)
//     = a[min((mK+j+1)*span_l, n) - 1] if (mK+j)*span_l < n and j < K-1, else MAX,
//     span_l = C * K^(L-1-l).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "params.h"

namespace bs {

template <class K>
__global__ void k_check_sorted(const K* __restrict__ a, uint64_t n, int* flag) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (a[i] > a[i + 1]) { atomicOr(flag, 1); return; }
    }
}

struct LevelBases { uint32_t base[kMaxLevels + 1]; };

template <class K>
__global__ void k_build_table(const K* __restrict__ a, uint64_t n, uint64_t s0, uint32_t nlev,
                              LevelBases lb, K* __restrict__ tab, uint64_t entries) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < entries;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t d = 0;
        while (d + 1 < nlev && lb.base[d + 1] <= e) ++d;
        const uint64_t k = e - lb.base[d];
        const uint64_t pos = n - 1 - (2 * k + 1) * (s0 >> d);
        tab[e] = a[pos];
    }
}

struct KaryMeta {
    uint64_t start[kMaxKaryLevels + 1];  // slot offset of level l (top-first, padded)
    uint64_t end[kMaxKaryLevels];        // start[l] + nodes_l * W (slots past it are padding)
    uint64_t span[kMaxKaryLevels];       // keys per child at level l
};

template <class K>
__global__ void k_build_kary(const K* __restrict__ a, uint64_t n, uint32_t Kf, uint32_t W, uint32_t L,
                             KaryMeta meta, K* __restrict__ sep, uint64_t slots) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < slots;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t l = 0;
        while (l + 1 < L && meta.start[l + 1] <= e) ++l;
        const uint64_t rel = e - meta.start[l];
        const uint64_t node = rel / W, j = rel % W;
        K v = KeyMax<K>::v;
        if (e < meta.end[l] && j + 1 < Kf) {
            const uint64_t child = node * Kf + j;
            const uint64_t span = meta.span[l];
            if (child * span < n) {
                uint64_t end = (child + 1) * span;
                if (end > n) end = n;
                v = a[end - 1];
            }
        }
        sep[e] = v;
    }
}

static unsigned grid_for(uint64_t work, unsigned threads) {
    uint64_t g = (work + threads - 1) / threads;
    if (g > 148ull * 64) g = 148ull * 64;
    if (g == 0) g = 1;
    return (unsigned)g;
}

cudaError_t build_check_sorted(int kb, const void* a, uint64_t n, int* d_flag, cudaStream_t s) {
    if (n < 2) return cudaSuccess;
    if (kb == 8) k_check_sorted<uint64_t><<<grid_for(n, 256), 256, 0, s>>>((const uint64_t*)a, n, d_flag);
    else k_check_sorted<uint32_t><<<grid_for(n, 256), 256, 0, s>>>((const uint32_t*)a, n, d_flag);
    return cudaGetLastError();
}

cudaError_t build_pinned_table(int kb, const void* a, uint64_t n, uint64_t s0, uint32_t nlev,
                               const uint32_t* base, void* tab, uint64_t entries, cudaStream_t s) {
    if (entries == 0) return cudaSuccess;
    LevelBases lb{};
    for (uint32_t d = 0; d <= nlev && d <= (uint32_t)kMaxLevels; ++d) lb.base[d] = base[d];
    if (kb == 8)
        k_build_table<uint64_t><<<grid_for(entries, 256), 256, 0, s>>>((const uint64_t*)a, n, s0, nlev, lb,
                                                                      (uint64_t*)tab, entries);
    else
        k_build_table<uint32_t><<<grid_for(entries, 256), 256, 0, s>>>((const uint32_t*)a, n, s0, nlev, lb,
                                                                      (uint32_t*)tab, entries);
    return cudaGetLastError();
}

cudaError_t build_kary_levels(int kb, const void* a, uint64_t n, uint32_t Kf, uint32_t C, uint32_t W,
                              uint32_t L, const uint64_t* lvl_base, const uint64_t* lvl_nodes,
                              void* sep, uint64_t slots, cudaStream_t s) {
    if (slots == 0 || L == 0) return cudaSuccess;
    KaryMeta meta{};
    for (uint32_t l = 0; l < L; ++l) {
        meta.start[l] = lvl_base[l];
        meta.end[l] = lvl_base[l] + lvl_nodes[l] * W;   // slots up to start[l+1] are MAX padding
        uint64_t span = C;
        for (uint32_t t = l + 1; t < L; ++t) span *= Kf;   // bottom level (l = L-1) spans C
        meta.span[l] = span;
    }
    meta.start[L] = slots;
    if (kb == 8)
        k_build_kary<uint64_t><<<grid_for(slots, 256), 256, 0, s>>>((const uint64_t*)a, n, Kf, W, L, meta,
                                                                    (uint64_t*)sep, slots);
    else
        k_build_kary<uint32_t><<<grid_for(slots, 256), 256, 0, s>>>((const uint32_t*)a, n, Kf, W, L, meta,
                                                                    (uint32_t*)sep, slots);
    return cudaGetLastError();
}

struct ImgMeta {
    uint64_t sep_base[kMaxKaryLevels];
    uint64_t start[kMaxKaryLevels + 1];   // cumulative image slots (node*(W+1)) per level
    uint32_t img_base[kMaxKaryLevels];
};

// Tiered shared-memory image: slot s of node m of level l -> word
// img_base[l] + m*(W+1) + s of each plane; s == W is padding.
template <class K, bool PAIR>
__global__ void k_build_img(const K* __restrict__ sep, uint32_t W, uint32_t L, ImgMeta meta, uint32_t* __restrict__ img,
                            uint64_t plane_words) {
    const uint64_t total = meta.start[L];
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t l = 0;
        while (l + 1 < L && meta.start[l + 1] <= e) ++l;
        const uint64_t rel = e - meta.start[l];
        const uint64_t node = rel / (W + 1), s = rel % (W + 1);
        const K v = (s < W) ? sep[meta.sep_base[l] + node * W + s] : KeyMax<K>::v;
        const uint64_t w = meta.img_base[l] + rel;
        if constexpr (PAIR) {
            reinterpret_cast<uint64_t*>(img)[w] = (uint64_t)v;
        } else if constexpr (sizeof(K) == 8) {
            img[w] = (uint32_t)((uint64_t)v >> 32);
            img[plane_words + w] = (uint32_t)v;
        } else {
            img[w] = (uint32_t)v;
        }
    }
}

cudaError_t build_kary_image(int kb, const void* sep, uint32_t W, uint32_t L, const uint64_t* lvl_base,
                              const uint64_t* lvl_nodes, const uint32_t* img_base, uint64_t plane_words,
                              void* img, bool pair64, cudaStream_t s) {
    if (L == 0) return cudaSuccess;
    ImgMeta meta;
    uint64_t acc = 0;
    for (uint32_t l = 0; l < L; ++l) {
        meta.sep_base[l] = lvl_base[l];
        meta.img_base[l] = img_base[l];
        meta.start[l] = acc;
        acc += lvl_nodes[l] * (W + 1);
    }
    meta.start[L] = acc;
    if (kb == 8 && pair64)
        k_build_img<uint64_t, true><<<grid_for(acc, 256), 256, 0, s>>>((const uint64_t*)sep, W, L, meta, (uint32_t*)img, plane_words);
    else if (kb == 8)
        k_build_img<uint64_t, false><<<grid_for(acc, 256), 256, 0, s>>>((const uint64_t*)sep, W, L, meta, (uint32_t*)img, plane_words);
    else
        k_build_img<uint32_t, false><<<grid_for(acc, 256), 256, 0, s>>>((const uint32_t*)sep, W, L, meta, (uint32_t*)img, plane_words);
    return cudaGetLastError();
}

// Flat pinned table in Eytzinger (BFS) order: slot k (1 <= k < 2^D) at depth
// d = floor(log2 k) holds sorted entry i = (2(k - 2^d) + 1) 2^(D-1-d) - 1;
// entry i < M = nodes - 1 is the max key of node i of the chosen K-ary level
// (span keys per node), the rest are MAX.  Slot 0 is unused.  Probes at depth
// d touch the contiguous slots [2^d, 2^(d+1)), so lanes spread over banks
// (a plain sorted array makes every lane of a halving step hit one bank).
// order-preserving 32-bit image of a u64 key (Index::flat_fbase / flat_fshift)
__device__ __forceinline__ uint32_t flat_image64(uint64_t x, uint64_t base, uint32_t sh) {
    if (x <= base) return 0u;
    const uint64_t d = (x - base) >> sh;
    return d > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)d;
}

template <class K>
__global__ void k_build_flat(const K* __restrict__ a, uint64_t n, uint64_t span, uint64_t M, uint32_t D,
                             uint32_t* __restrict__ f32, uint64_t* __restrict__ f64, uint64_t fbase, uint32_t fshift) {
    const uint64_t slots = 1ull << D;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < slots;
         k += (uint64_t)gridDim.x * blockDim.x) {
        K v = KeyMax<K>::v;
        if (k > 0) {
            const uint32_t d = 63 - __clzll((long long)k);
            const uint64_t i = ((2 * (k - (1ull << d)) + 1) << (D - 1 - d)) - 1;
            if (i < M) {
                uint64_t end = (i + 1) * span;
                if (end > n) end = n;
                v = a[end - 1];
            }
        }
        if constexpr (sizeof(K) == 8) {
            f32[k] = flat_image64((uint64_t)v, fbase, fshift);
            f64[k] = (uint64_t)v;
        } else {
            f32[k] = (uint32_t)v;
        }
    }
}

cudaError_t build_flat_table(int kb, const void* a, uint64_t n, uint64_t span, uint64_t M, uint32_t D,
                             void* flat32, void* flat64, uint64_t fbase, uint32_t fshift, cudaStream_t s) {
    const uint64_t slots = 1ull << D;
    if (kb == 8)
        k_build_flat<uint64_t><<<grid_for(slots, 256), 256, 0, s>>>((const uint64_t*)a, n, span, M, D,
                                                                    (uint32_t*)flat32, (uint64_t*)flat64, fbase, fshift);
    else
        k_build_flat<uint32_t><<<grid_for(slots, 256), 256, 0, s>>>((const uint32_t*)a, n, span, M, D,
                                                                    (uint32_t*)flat32, nullptr, 0, 0);
    return cudaGetLastError();
}

// the flat level's node image in the flat table's 32-bit image (u64: from the
// hi / lo planes of the tiered image; u32: the plane as is)
__global__ void k_flat_level_image(const uint32_t* __restrict__ hi, const uint32_t* __restrict__ lo, uint64_t words,
                                   uint64_t fbase, uint32_t fshift, uint32_t* __restrict__ out) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x)
        out[w] = lo ? flat_image64(((uint64_t)hi[w] << 32) | lo[w], fbase, fshift) : hi[w];
}

cudaError_t build_flat_level_image(const uint32_t* hi, const uint32_t* lo, uint64_t words, uint64_t fbase,
                                   uint32_t fshift, uint32_t* out, cudaStream_t s) {
    if (!words) return cudaSuccess;
    k_flat_level_image<<<grid_for(words, 256), 256, 0, s>>>(hi, lo, words, fbase, fshift, out);
    return cudaGetLastError();
}

cudaError_t build_sort_keys(int kb, const void* in, void* out, uint64_t n, cudaStream_t s) {
    size_t tmp_bytes = 0;
    cudaError_t e;
    if (kb == 8)
        e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, (const uint64_t*)in, (uint64_t*)out, (int64_t)n, 0, 64, s);
    else
        e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, (const uint32_t*)in, (uint32_t*)out, (int64_t)n, 0, 32, s);
    if (e != cudaSuccess) return e;
    void* tmp = nullptr;
    e = cudaMallocAsync(&tmp, tmp_bytes, s);
    if (e != cudaSuccess) return e;
    if (kb == 8)
        e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, (const uint64_t*)in, (uint64_t*)out, (int64_t)n, 0, 64, s);
    else
        e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, (const uint32_t*)in, (uint32_t*)out, (int64_t)n, 0, 32, s);
    cudaFreeAsync(tmp, s);
    return e;
}

}  // namespace bs
