// ubench_shfl.cu — which warp-level primitives consume L1 data-pipe (shared) wavefronts?
// Each kernel runs N iterations of one primitive; profile with
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,gpu__time_duration.sum
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_shfl32(uint32_t* o, int n) {
    uint32_t v = threadIdx.x;
    for (int i = 0; i < n; ++i) v += __shfl_xor_sync(0xFFFFFFFFu, v, 1 + (i & 3));
    if (v == 0x12345) *o = v;
}
__global__ void k_shfl_idx(uint32_t* o, int n) {
    uint32_t v = threadIdx.x;
    for (int i = 0; i < n; ++i) v += __shfl_sync(0xFFFFFFFFu, v, (threadIdx.x * 5 + i) & 31);
    if (v == 0x12345) *o = v;
}
__global__ void k_vote(uint32_t* o, int n) {
    uint32_t v = threadIdx.x;
    for (int i = 0; i < n; ++i) v += __popc(__ballot_sync(0xFFFFFFFFu, (v >> (i & 7)) & 1));
    if (v == 0x12345) *o = v;
}
__global__ void k_redux(uint32_t* o, int n) {
    uint32_t v = threadIdx.x;
    for (int i = 0; i < n; ++i) v += __reduce_add_sync(0xFFFFFFFFu, v & 15);
    if (v == 0x12345) *o = v;
}
__global__ void k_redux_group(uint32_t* o, int n) {   // 8 disjoint groups of 4 lanes
    uint32_t v = threadIdx.x;
    const uint32_t gm = 0xFu << ((threadIdx.x & 31) & ~3u);
    for (int i = 0; i < n; ++i) v += __reduce_add_sync(gm, v & 15);
    if (v == 0x12345) *o = v;
}
__global__ void k_lds(uint32_t* o, int n) {
    __shared__ uint32_t s[1024];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    uint32_t v = threadIdx.x;
    for (int i = 0; i < n; ++i) v = s[(v + i) & 1023] + 1;   // conflict-free-ish broadcast pattern varies
    if (v == 0x12345) *o = v;
}
__global__ void k_lds_pred_off(uint32_t* o, int n, uint32_t never) {
    __shared__ uint32_t s[1024];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    uint32_t v = threadIdx.x;
    for (int i = 0; i < n; ++i) {
        v += 3;
        if (v == never) v = s[v & 1023];   // predicated-off shared load
    }
    if (v == 0x12345) *o = v;
}

int main() {
    uint32_t* o;
    cudaMalloc(&o, 4);
    const int n = 4096, B = 148 * 4, T = 256;
    k_shfl32<<<B, T>>>(o, n);
    k_shfl_idx<<<B, T>>>(o, n);
    k_vote<<<B, T>>>(o, n);
    k_redux<<<B, T>>>(o, n);
    k_redux_group<<<B, T>>>(o, n);
    k_lds<<<B, T>>>(o, n);
    k_lds_pred_off<<<B, T>>>(o, n, 0xFFFFFFFFu);
    cudaDeviceSynchronize();
    printf("warp-ops per kernel: %d\n", B * (T / 32) * n);
    return 0;
}
