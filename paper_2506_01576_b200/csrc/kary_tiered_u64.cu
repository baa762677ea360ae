// kary_tiered_u64.cu — u64 instantiations of the tiered K-ary kernel (kary_tiered.cuh).
#include "kary_tiered.cuh"

namespace bs {
template cudaError_t dispatch_tiered<uint64_t>(const void*, const void*, uint64_t, void*, uint32_t, uint32_t, uint32_t,
                                               uint32_t, uint32_t, bool, bool, Grid, uint32_t, cudaStream_t, bool*);
}  // namespace bs
