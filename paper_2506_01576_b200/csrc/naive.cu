// naive.cu — Listing 1: one thread per lookup, dynamic grid.
//
// This is the in-repo baseline the optimised kernels are measured against
// (BASELINE.md §2): scalar loads, no cache hints, no shared memory.  The only
// additions to Listing 1 are reading R1 (halve every iteration), tracking the
// value of the last taken probe so the result can be encoded (hit/miss,
// reading R3), and 64-bit offsets.
#include "common.cuh"
#include "params.h"

namespace bs {

template <class K, class O>
__global__ void k_naive(const K* __restrict__ a, uint64_t n, const K* __restrict__ q, uint64_t m,
                        O* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;  // TID
    if (i >= m) return;
    const K lookup = q[i];                       // l.10  lookup = lookups[TID]
    uint64_t offset = n - 1;                     // l.11  offset = len(sorted_keys) - 1
    uint64_t step = lpow2(n);                    // l.12  step = LPOW2(len(sorted_keys))
    K v = a[n - 1];                              // value at `offset` (footnote 1)
    while (step > 0) {                           // l.2
        if (step <= offset) {                    // l.3
            const K x = a[offset - step];
            if (x >= lookup) {                   // l.4
                offset -= step;                  // l.5
                v = x;
            }
        }
        step >>= 1;                              // l.6 (reading R1: every iteration)
    }
    out[i] = encode<O>(offset, v, lookup, n);    // l.13 results[TID] = offset (+ miss bit)
}

cudaError_t launch_naive(int kb, int ob, const void* a, uint64_t n, const void* q, uint64_t m,
                         void* out, uint32_t threads, cudaStream_t s) {
    if (threads == 0) threads = 256;
    const uint64_t blocks = (m + threads - 1) / threads;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const dim3 g((unsigned)blocks), b(threads);
    if (kb == 8 && ob == 8)
        k_naive<uint64_t, uint64_t><<<g, b, 0, s>>>((const uint64_t*)a, n, (const uint64_t*)q, m, (uint64_t*)out);
    else if (kb == 8 && ob == 4)
        k_naive<uint64_t, uint32_t><<<g, b, 0, s>>>((const uint64_t*)a, n, (const uint64_t*)q, m, (uint32_t*)out);
    else if (kb == 4 && ob == 8)
        k_naive<uint32_t, uint64_t><<<g, b, 0, s>>>((const uint32_t*)a, n, (const uint32_t*)q, m, (uint64_t*)out);
    else
        k_naive<uint32_t, uint32_t><<<g, b, 0, s>>>((const uint32_t*)a, n, (const uint32_t*)q, m, (uint32_t*)out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace bs
