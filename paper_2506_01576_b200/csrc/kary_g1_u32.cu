// kary_g1_u32.cu — u32 instantiations of the thread-per-lookup K-ary kernel (kary_g1.cuh) + launcher.
#include "kary_g1.cuh"

namespace bs {
template cudaError_t dispatch_g1<uint32_t>(const void*, const void*, uint64_t, void*, uint32_t, uint32_t, uint32_t,
                                           uint32_t, uint32_t, uint32_t, bool, Grid, uint32_t, cudaStream_t, bool*);

cudaError_t launch_kary_g1(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                           uint32_t threads, uint32_t W, uint32_t GL, uint32_t IL, uint32_t T, bool flat, Grid grid, uint32_t smem,
                           cudaStream_t s, bool* uns) {
    *uns = false;
    if (kb == 8) return dispatch_g1<uint64_t>(params, q, m, out, (uint32_t)ob, threads, W, GL, IL, T, flat, grid, smem, s, uns);
    return dispatch_g1<uint32_t>(params, q, m, out, (uint32_t)ob, threads, W, GL, IL, T, flat, grid, smem, s, uns);
}
}  // namespace bs
