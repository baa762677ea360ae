// ubench_gather2.cu — how many random G-byte reads per second B200's HBM3e
// serves, and (under ncu) how many DRAM bytes each one costs.  Round-2 fix of
// ubench_gather.cu: addresses are masked into a power-of-two buffer (the
// 64-bit `% nunits` made the old G/s columns compute-bound), and every access
// is made of 256-bit loads (sm_100 LDG.E.ENL2.256), as the lookup kernels do.
//
// Layouts of one G-byte access:
//   T  one thread issues all G/32 loads (thread-per-lookup leaf)
//   L  G/32 consecutive lanes issue one 32-B load each (lane-group leaf)
// Optional stream: each access also reads 8 B and writes 8 B sequentially
// (query in, result out), as one lookup does.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_gather2 ubench_gather2.cu
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

__device__ __forceinline__ void ld32(const uint64_t* p, uint64_t pol, uint64_t* x) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=l"(x[0]), "=l"(x[1]), "=l"(x[2]), "=l"(x[3]) : "l"(p), "l"(pol));
}

template <int G, int ILP, bool LANES, bool STREAM>
__global__ void __launch_bounds__(256) gather(const uint64_t* __restrict__ buf, uint64_t mask_units, int iters,
                                              const uint64_t* __restrict__ qin, uint64_t* __restrict__ qout,
                                              uint64_t* sink, int first) {
    constexpr int NL = G / 32;                  // 256-bit loads per access
    constexpr int GL = LANES ? NL : 1;          // lanes per access
    const uint32_t lane = threadIdx.x & 31;
    uint64_t pol;
    if (first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t x[ILP][LANES ? 4 : NL * 4];
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            // one address per access: lanes of a group share it (group leader's hash)
            const uint64_t gid = LANES ? (tid / GL) : tid;
            const uint64_t u = mix(gid * 0x9E3779B97F4A7C15ull + (uint64_t)it * ILP + i) & mask_units;
            const uint64_t* p = buf + u * (G / 8);
            if constexpr (LANES) {
                ld32(p + (lane % GL) * 4, pol, x[i]);
            } else {
#pragma unroll
                for (int j = 0; j < NL; ++j) ld32(p + j * 4, pol, &x[i][j * 4]);
            }
        }
        if constexpr (STREAM) {
            // per access: 8 B in, 8 B out (coalesced), like one lookup's query and result
            const uint64_t base = ((uint64_t)it * nthr + tid) * ILP / (LANES ? GL : 1);
#pragma unroll
            for (int i = 0; i < ILP / (LANES ? GL : 1) + (LANES && ILP < GL ? 1 : 0); ++i) {
                const uint64_t o = (base + i) & ((1ull << 27) - 1);
                uint64_t v;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(qin + o), "l"(pol));
                acc += v;
                asm volatile("st.global.L1::no_allocate.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(qout + o), "l"(acc), "l"(pol) : "memory");
            }
        }
#pragma unroll
        for (int i = 0; i < ILP; ++i)
#pragma unroll
            for (int j = 0; j < (LANES ? 4 : NL * 4); ++j) acc += x[i][j];
    }
    if (acc == 0x12345) *sink = acc;
}

template <int G, int ILP, bool LANES, bool STREAM>
void run(const uint64_t* buf, uint64_t bytes, int blocks, int iters, const uint64_t* qin, uint64_t* qout,
         uint64_t* sink, int first) {
    const uint64_t units = bytes / G;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<G, ILP, LANES, STREAM><<<blocks, 256>>>(buf, units - 1, 2, qin, qout, sink, first);
    cudaEventRecord(a);
    gather<G, ILP, LANES, STREAM><<<blocks, 256>>>(buf, units - 1, iters, qin, qout, sink, first);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    constexpr int GL = LANES ? G / 32 : 1;
    const double acc = (double)blocks * 256 / GL * iters * ILP;
    printf("{\"bytes\": %llu, \"gran\": %d, \"ilp\": %d, \"lanes\": %d, \"stream\": %d, \"evict_first\": %d, "
           "\"blocks\": %d, \"ms\": %.4f, \"G_access_per_s\": %.3f, \"useful_GBps\": %.1f}\n",
           (unsigned long long)bytes, G, ILP, LANES ? 1 : 0, STREAM ? 1 : 0, first, blocks, ms, acc / ms / 1e6,
           acc * G / ms / 1e6);
    fflush(stdout);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}

int main(int argc, char** argv) {
    const uint64_t maxb = 8ull << 30;
    uint64_t *buf, *sink, *qin, *qout;
    if (cudaMalloc(&buf, maxb) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&sink, 8);
    cudaMalloc(&qin, 1ull << 30);
    cudaMalloc(&qout, 1ull << 30);
    cudaMemset(buf, 1, maxb);
    cudaMemset(qin, 2, 1ull << 30);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int only = argc > 1 ? atoi(argv[1]) : -1;   // -1 = full table; k = one row (for ncu)
    const int blocks = sms * 8;
    int row = 0;
#define ROW(...) if (only < 0 || only == row) { __VA_ARGS__; } ++row;
    for (uint64_t bytes : {32ull << 20, 512ull << 20, 8ull << 30}) {
        ROW((run<32, 8, false, false>(buf, bytes, blocks, 16, qin, qout, sink, 1)))
        ROW((run<64, 8, false, false>(buf, bytes, blocks, 16, qin, qout, sink, 1)))
        ROW((run<128, 4, false, false>(buf, bytes, blocks, 16, qin, qout, sink, 1)))
        ROW((run<64, 8, true, false>(buf, bytes, blocks, 16, qin, qout, sink, 1)))
        ROW((run<128, 8, true, false>(buf, bytes, blocks, 16, qin, qout, sink, 1)))
        ROW((run<64, 8, false, true>(buf, bytes, blocks, 16, qin, qout, sink, 1)))
        ROW((run<128, 8, true, true>(buf, bytes, blocks, 16, qin, qout, sink, 1)))
        ROW((run<64, 8, false, false>(buf, bytes, blocks, 16, qin, qout, sink, 0)))
        ROW((run<128, 4, false, false>(buf, bytes, blocks, 16, qin, qout, sink, 0)))
    }
    printf("{\"rows\": %d}\n", row);
    return 0;
}
