// ubench_flavors.cu — what one random 32-B read costs on B200, per PTX load
// flavour.  ubench_gather2.cu measured only ld.global.nc (the texture path):
// every random 32-B read moved ~4 L2 sectors to the SM and ~107-127 DRAM
// bytes.  This table asks whether that is the DRAM atom or the load path:
// the same random 32-B accesses (one thread each, 8 in flight) issued as
//
//   0  ld.global.nc.L1::no_allocate.v4.u64   (the kernels' current form)
//   1  ld.global.nc.v4.u64                   (L1-allocating texture path)
//   2  ld.global.cg.v4.u64                   (cache at L2, not L1)
//   3  ld.global.cv.v4.u64                   (volatile: fetch again)
//   4  ld.relaxed.gpu.global.v4.u64          (memory-model load)
//   5  ld.global.L1::no_allocate.v4.u64      (coherent path, no L1 allocation)
//   6  ld.global.nc.L1::no_allocate.v2.u64 x2 (two 16-B loads)
//   7  ld.global.cg.v2.u64 x2
//
// with the L2 fetch granularity limit at its default or 32 B (argv[2]), over
// a 32 MB (L2-resident) and an 8 GB buffer.  Run one row under ncu:
//   ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,... ./ubench_flavors ROW [fetch32]
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_flavors ubench_flavors.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int F>
__device__ __forceinline__ void ld32(const uint64_t* p, uint64_t* x) {
    if constexpr (F == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p));
    else if constexpr (F == 1)
        asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p));
    else if constexpr (F == 2)
        asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p));
    else if constexpr (F == 3)
        asm volatile("ld.global.cv.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p));
    else if constexpr (F == 4)
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p));
    else if constexpr (F == 5)
        asm volatile("ld.global.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p));
    else if constexpr (F == 6) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(x[0]), "=l"(x[1]) : "l"(p));
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(x[2]), "=l"(x[3]) : "l"(p + 2));
    } else {
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(x[0]), "=l"(x[1]) : "l"(p));
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(x[2]), "=l"(x[3]) : "l"(p + 2));
    }
}

template <int F, int ILP>
__global__ void __launch_bounds__(256) gather(const uint64_t* __restrict__ buf, uint64_t mask_units, int iters,
                                              uint64_t* sink) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t x[ILP][4];
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            const uint64_t u = mix(tid * 0x9E3779B97F4A7C15ull + (uint64_t)it * ILP + i) & mask_units;
            ld32<F>(buf + u * 4, x[i]);
        }
#pragma unroll
        for (int i = 0; i < ILP; ++i) acc += x[i][0] ^ x[i][1] ^ x[i][2] ^ x[i][3];
    }
    if (acc == 0x12345) *sink = acc;
}

template <int F>
void run(const uint64_t* buf, uint64_t bytes, int blocks, int iters, uint64_t* sink, int fetch) {
    constexpr int ILP = 8;
    const uint64_t units = bytes / 32;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<F, ILP><<<blocks, 256>>>(buf, units - 1, 2, sink);
    cudaEventRecord(a);
    gather<F, ILP><<<blocks, 256>>>(buf, units - 1, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double acc = (double)blocks * 256 * iters * ILP;
    printf("{\"flavor\": %d, \"bytes\": %llu, \"fetch_limit\": %d, \"ms\": %.4f, \"accesses\": %.0f, "
           "\"G_access_per_s\": %.3f, \"err\": \"%s\"}\n",
           F, (unsigned long long)bytes, fetch, ms, acc, acc / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}

int main(int argc, char** argv) {
    const uint64_t maxb = 8ull << 30;
    uint64_t *buf, *sink;
    if (cudaMalloc(&buf, maxb) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, maxb);
    const int only = argc > 1 ? atoi(argv[1]) : -1;     // -1 = all rows; k = one row (for ncu)
    const int fetch = argc > 2 ? atoi(argv[2]) : 0;     // 0 = default L2 fetch granularity
    if (fetch) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)fetch);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8;
    int row = 0;
#define ROW(F) if (only < 0 || only == row) { run<F>(buf, bytes, blocks, 16, sink, (int)got); } ++row;
    for (uint64_t bytes : {32ull << 20, 8ull << 30}) {
        ROW(0) ROW(1) ROW(2) ROW(3) ROW(4) ROW(5) ROW(6) ROW(7)
    }
    printf("{\"rows\": %d}\n", row);
    return 0;
}
