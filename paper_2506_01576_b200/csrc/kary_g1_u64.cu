// kary_g1_u64.cu — u64 instantiations of the thread-per-lookup K-ary kernel (kary_g1.cuh).
#include "kary_g1.cuh"

namespace bs {
template cudaError_t dispatch_g1<uint64_t>(const void*, const void*, uint64_t, void*, uint32_t, uint32_t, uint32_t,
                                           uint32_t, uint32_t, uint32_t, bool, Grid, uint32_t, cudaStream_t, bool*);
}  // namespace bs
