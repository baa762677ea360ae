// ubench_gather.cu — random-gather throughput of B200 HBM3e / L2 at a given
// access granularity and load flavour (the roofline denominator for a random
// lookup: how many independent random accesses per second the memory system
// serves, and how many DRAM bytes each one really costs).
//
// Each thread issues ILP independent loads of G bytes at random G-aligned
// offsets in a buffer of B bytes (counter-based hash addresses, no dependency
// chain), for ITER rounds.  Flavours:
//   0 ld.global.nc                      (L1-allocating read-only path)
//   1 ld.global.nc.L1::no_allocate      (no L1 line fill)
//   2 ld.global.cg                      (cache at L2 only)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_gather ubench_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int F>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
    uint4 r;
    if (F == 0)
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (F == 1)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
template <int F>
__device__ __forceinline__ uint64_t ld8(const uint64_t* p) {
    uint64_t r;
    if (F == 0) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(r) : "l"(p));
    else if (F == 1) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(p));
    else asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}

template <int G, int ILP, int F>
__global__ void gather(const uint4* __restrict__ buf, uint64_t nunits, int iters, uint64_t* sink) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    constexpr int V = G / 16 > 0 ? G / 16 : 1;   // uint4 per access
    for (int it = 0; it < iters; ++it) {
        uint4 v[ILP][V];
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            const uint64_t u = mix(tid * 1315423911ull + (uint64_t)it * ILP + i) % nunits;
            if (G >= 16) {
#pragma unroll
                for (int j = 0; j < V; ++j) v[i][j] = ld16<F>(buf + u * V + j);
            } else {
                const uint64_t x = ld8<F>(reinterpret_cast<const uint64_t*>(buf) + u);
                v[i][0] = make_uint4((uint32_t)x, (uint32_t)(x >> 32), 0, 0);
            }
        }
#pragma unroll
        for (int i = 0; i < ILP; ++i)
#pragma unroll
            for (int j = 0; j < V; ++j) acc += v[i][j].x ^ v[i][j].w;
    }
    if (acc == 0x12345) *sink = acc;
}

template <int G, int ILP, int F>
void run(const uint4* buf, uint64_t bytes, int blocks, int threads, int iters, uint64_t* sink) {
    const uint64_t nunits = bytes / (G >= 16 ? G : 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<G, ILP, F><<<blocks, threads>>>(buf, nunits, 2, sink);
    cudaEventRecord(a);
    gather<G, ILP, F><<<blocks, threads>>>(buf, nunits, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double acc = (double)blocks * threads * iters * ILP;
    printf("{\"bytes\": %llu, \"gran\": %d, \"ilp\": %d, \"flavour\": %d, \"threads\": %d, \"blocks\": %d, "
           "\"G_access_per_s\": %.3f, \"useful_GBps\": %.1f}\n",
           (unsigned long long)bytes, G, ILP, F, threads, blocks, acc / ms / 1e6, acc * G / ms / 1e6);
    fflush(stdout);
}

int main(int argc, char** argv) {
    const uint64_t maxb = 8ull << 30;
    uint4* buf;
    uint64_t* sink;
    if (cudaMalloc(&buf, maxb) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, maxb);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t gran = 0;
    cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
    printf("{\"default_l2_fetch_granularity\": %zu}\n", gran);
    const int fetch = argc > 1 ? atoi(argv[1]) : 0;
    if (fetch) {
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, fetch);
        cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
        printf("{\"l2_fetch_granularity\": %zu}\n", gran);
    }
    for (uint64_t bytes : {32ull << 20, 512ull << 20, 8ull << 30}) {
        run<8, 8, 0>(buf, bytes, sms * 8, 256, 64, sink);
        run<8, 8, 1>(buf, bytes, sms * 8, 256, 64, sink);
        run<8, 8, 2>(buf, bytes, sms * 8, 256, 64, sink);
        run<32, 8, 1>(buf, bytes, sms * 8, 256, 64, sink);
        run<32, 8, 2>(buf, bytes, sms * 8, 256, 64, sink);
        run<64, 4, 1>(buf, bytes, sms * 8, 256, 64, sink);
        run<128, 2, 1>(buf, bytes, sms * 8, 256, 64, sink);
        run<8, 16, 1>(buf, bytes, sms * 8, 256, 32, sink);
    }
    return 0;
}
