// kary_tiered_u32.cu — u32 instantiations of the tiered K-ary kernel (kary_tiered.cuh).
#include "kary_tiered.cuh"

namespace bs {
template cudaError_t dispatch_tiered<uint32_t>(const void*, const void*, uint64_t, void*, uint32_t, uint32_t, uint32_t,
                                               uint32_t, uint32_t, bool, bool, Grid, uint32_t, cudaStream_t, bool*);

cudaError_t launch_kary_tiered(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                               uint32_t threads, uint32_t W, uint32_t R, uint32_t I, bool pair64, bool pipe, Grid grid,
                               uint32_t smem, cudaStream_t s, bool* uns) {
    *uns = false;
    if (kb == 8) return dispatch_tiered<uint64_t>(params, q, m, out, (uint32_t)ob, threads, W, R, I, pair64, pipe, grid, smem, s, uns);
    return dispatch_tiered<uint32_t>(params, q, m, out, (uint32_t)ob, threads, W, R, I, pair64, pipe, grid, smem, s, uns);
}
}  // namespace bs
