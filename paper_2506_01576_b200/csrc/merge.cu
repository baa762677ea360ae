// merge.cu — batch inserts and deletes (§6 outlook,
// "the cost of performing batch-wise updates" — the paper gives no
// method).  bs_erase: flag every key of the array that occurs in the sorted
// delete set (binary search per key), compact the survivors with
// cub::DeviceSelect::Flagged into a buffer the new index adopts, rebuild.
//
// An index is immutable (its auxiliary levels are copies derived from the
// sorted array), so a batch of inserts produces a NEW index over the multiset
// union: sort the delta (CUB radix sort, the library's build sort), merge it
// with the old sorted array by a merge-path kernel (each thread binary-searches
// its diagonal split, then merges its slice; ties take the old key first,
// which is immaterial for keys-only data), and build the new index's pinned
// table / separator levels / images over the merged array with the same
// layout.  Results on the new index are those of the oracle on
// sort(a ++ delta) (tests/test_gpu_merge.py).
#include <cstring>

#include <cub/device/device_select.cuh>

#include "index.h"

namespace bs {

constexpr uint32_t kMergePer = 16;   // outputs per thread

template <class K>
__global__ void __launch_bounds__(256) k_merge_path(const K* __restrict__ a, uint64_t na, const K* __restrict__ b,
                                                    uint64_t nb, K* __restrict__ out) {
    const uint64_t total = na + nb;
    const uint64_t diag = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kMergePer;
    if (diag >= total) return;
    // split: i elements from a, diag - i from b, with a[i-1] <= b[diag-i] (a first on ties)
    uint64_t lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] <= b[diag - mid - 1]) lo = mid + 1;
        else hi = mid;
    }
    uint64_t i = lo, j = diag - lo;
    const uint64_t end = diag + kMergePer < total ? diag + kMergePer : total;
    for (uint64_t o = diag; o < end; ++o) {
        const bool take_a = j >= nb || (i < na && a[i] <= b[j]);
        out[o] = take_a ? a[i++] : b[j++];
    }
}

static cudaError_t launch_merge(uint32_t kb, const void* a, uint64_t na, const void* b, uint64_t nb, void* out,
                                cudaStream_t s) {
    const uint64_t threads = (na + nb + kMergePer - 1) / kMergePer;
    const uint64_t blocks = (threads + 255) / 256;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    if (kb == 8)
        k_merge_path<uint64_t><<<(unsigned)blocks, 256, 0, s>>>((const uint64_t*)a, na, (const uint64_t*)b, nb,
                                                               (uint64_t*)out);
    else
        k_merge_path<uint32_t><<<(unsigned)blocks, 256, 0, s>>>((const uint32_t*)a, na, (const uint32_t*)b, nb,
                                                               (uint32_t*)out);
    return cudaGetLastError();
}

// keep[i] = a[i] is not in the sorted delete set d[0..m) (binary search)
template <class K>
__global__ void k_erase_flags(const K* __restrict__ a, uint64_t n, const K* __restrict__ d, uint64_t m,
                              uint8_t* __restrict__ keep) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const K x = a[i];
        uint64_t lo = 0, hi = m;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (d[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        keep[i] = (lo < m && d[lo] == x) ? 0 : 1;
    }
}

template <class K>
static cudaError_t erase_compact(const K* a, uint64_t n, const K* d, uint64_t m, K* out, uint64_t* d_count,
                                 cudaStream_t s) {
    uint8_t* keep = nullptr;
    cudaError_t e = cudaMallocAsync(&keep, n, s);
    if (e != cudaSuccess) return e;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    k_erase_flags<K><<<(unsigned)blocks, 256, 0, s>>>(a, n, d, m, keep);
    e = cudaGetLastError();
    size_t tmp_bytes = 0;
    if (e == cudaSuccess) e = cub::DeviceSelect::Flagged(nullptr, tmp_bytes, a, keep, out, d_count, (int64_t)n, s);
    void* tmp = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tmp_bytes, s);
    if (e == cudaSuccess) e = cub::DeviceSelect::Flagged(tmp, tmp_bytes, a, keep, out, d_count, (int64_t)n, s);
    if (tmp) cudaFreeAsync(tmp, s);
    cudaFreeAsync(keep, s);
    return e;
}

}  // namespace bs

using namespace bs;

extern "C" {

int bs_merge(const void* idx, const void* delta_keys, uint64_t m, int delta_sorted, void** out_idx) {
    if (!idx || !out_idx) return fail(BS_ERR_INVALID, "bs_merge: NULL");
    *out_idx = nullptr;
    const Index* ix = (const Index*)idx;
    if (ix->dist || ix->peer) return fail(BS_ERR_UNSUPPORTED, "bs_merge: multi-GPU indexes are not merged (merge each shard)");
    if (m && !delta_keys) return fail(BS_ERR_INVALID, "bs_merge: delta_keys is NULL with m > 0");
    bs_layout lay = ix->layout;
    lay.cache_hints = ix->hints_requested;
    lay.kary_mode = ix->kary_mode_requested;
    lay.leaf_chunk = ix->leaf_chunk_requested;
    lay.input_sorted = 1;
    const uint64_t total = ix->n + m;
    if (lay.out_bytes == 4 && total >= (1ull << 31)) return fail(BS_ERR_INVALID, "bs_merge: out_bytes = 4 requires n + m < 2^31");
    if (m == 0) return bs_build(ix->d_keys, ix->n, &lay, out_idx);
    const uint32_t kb = ix->kb;
    cudaStream_t s = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail_cuda(e, "bs_merge: stream");
    void* sorted = nullptr;
    void* merged = nullptr;
    int rc = BS_OK;
    // the new index adopts this buffer: bs_build's layout (n keys + 256 pad keys + 16 B)
    e = cudaMalloc(&merged, total * kb + 256 * kb + 16);
    if (e == cudaSuccess && !delta_sorted) {
        e = cudaMallocAsync(&sorted, m * kb, s);
        if (e == cudaSuccess) e = build_sort_keys((int)kb, delta_keys, sorted, m, s);
    }
    if (e == cudaSuccess) e = launch_merge(kb, ix->d_keys, ix->n, delta_sorted ? delta_keys : sorted, m, merged, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail_cuda(e, "bs_merge: sort / merge");
    if (sorted) cudaFreeAsync(sorted, s);
    cudaStreamSynchronize(s);
    // bs_build re-checks ascending order (a delta_sorted = 1 that is not sorted
    // -> BS_ERR_NOT_SORTED) and adopts `merged` (freed with the index, or by
    // bs_build itself on failure)
    if (rc == BS_OK) {
        t_adopt_keys = merged;
        rc = bs_build(merged, total, &lay, out_idx);
        if (t_adopt_keys) {   // bs_build returned before taking the buffer (argument check)
            t_adopt_keys = nullptr;
            cudaFree(merged);
        }
    } else if (merged) {
        cudaFree(merged);
    }
    cudaStreamDestroy(s);
    return rc;
}

}  // extern "C"


extern "C" {

int bs_erase(const void* idx, const void* del_keys, uint64_t m, int del_sorted, void** out_idx) {
    if (!idx || !out_idx) return fail(BS_ERR_INVALID, "bs_erase: NULL");
    *out_idx = nullptr;
    const Index* ix = (const Index*)idx;
    if (ix->dist || ix->peer) return fail(BS_ERR_UNSUPPORTED, "bs_erase: multi-GPU indexes are not edited (edit each shard)");
    if (m && !del_keys) return fail(BS_ERR_INVALID, "bs_erase: del_keys is NULL with m > 0");
    bs_layout lay = ix->layout;
    lay.cache_hints = ix->hints_requested;
    lay.kary_mode = ix->kary_mode_requested;
    lay.leaf_chunk = ix->leaf_chunk_requested;
    lay.input_sorted = 1;
    if (m == 0) return bs_build(ix->d_keys, ix->n, &lay, out_idx);
    const uint32_t kb = ix->kb;
    cudaStream_t s = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail_cuda(e, "bs_erase: stream");
    void* sorted = nullptr;
    void* kept = nullptr;
    uint64_t* d_count = nullptr;
    uint64_t count = 0;
    int rc = BS_OK;
    // the new index adopts this buffer: bs_build's layout (n keys + 256 pad keys + 16 B)
    e = cudaMalloc(&kept, ix->n * kb + 256 * kb + 16);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&d_count, sizeof(uint64_t), s);
    if (e == cudaSuccess && !del_sorted) {
        e = cudaMallocAsync(&sorted, m * kb, s);
        if (e == cudaSuccess) e = build_sort_keys((int)kb, del_keys, sorted, m, s);
    }
    const void* d = del_sorted ? del_keys : sorted;
    if (e == cudaSuccess)
        e = kb == 8 ? erase_compact<uint64_t>((const uint64_t*)ix->d_keys, ix->n, (const uint64_t*)d, m,
                                               (uint64_t*)kept, d_count, s)
                    : erase_compact<uint32_t>((const uint32_t*)ix->d_keys, ix->n, (const uint32_t*)d, m,
                                               (uint32_t*)kept, d_count, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&count, d_count, sizeof count, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail_cuda(e, "bs_erase: sort / flag / compact");
    if (sorted) cudaFreeAsync(sorted, s);
    if (d_count) cudaFreeAsync(d_count, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc == BS_OK && count == 0) rc = fail(BS_ERR_INVALID, "bs_erase: every key would be erased (an index needs n >= 1)");
    // (an unsorted delete set claimed sorted only misses deletions; the result stays ascending)
    if (rc == BS_OK) {
        t_adopt_keys = kept;
        rc = bs_build(kept, count, &lay, out_idx);
        if (t_adopt_keys) {
            t_adopt_keys = nullptr;
            cudaFree(kept);
        }
    } else if (kept) {
        cudaFree(kept);
    }
    return rc;
}

}  // extern "C"
