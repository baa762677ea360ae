// peer_sync.cuh — device-side signalling for the fused peer-memory routing
// path (peer.cu, the g1 lookup epilogue).  Ranks exchange queries and results
// by plain stores into each other's IPC-mapped windows (NVLink / NVSwitch P2P
// on a multi-GPU box) and publish completion with monotonic 64-bit counters:
// every rank adds 1 to every rank's counter once per call, so call t is
// complete at a rank when its counter reaches t * P.  Writers fence at system
// scope before the release-add; readers spin with acquire loads.
#pragma once
#include <cstdint>

namespace bs {

constexpr unsigned kPeerErrOverflow = 1u;   // a receive window was full (queries dropped)
constexpr unsigned kPeerErrTimeout = 2u;    // a wait gave up (a peer never signalled)
constexpr unsigned long long kPeerWaitNs = 20ull * 1000 * 1000 * 1000;   // 20 s (default)

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_sys_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin (one thread) until *p >= target; bounded so a dead peer cannot hang
// the GPU: after the limit the error bit is set and the wait returns.  The
// limit in ms sits in the word after the error bits (PeerCtl::wait_ms; 0 =
// kPeerWaitNs).
__device__ __forceinline__ void peer_wait_ge(const unsigned long long* p, unsigned long long target, unsigned* err) {
    if (ld_acquire_sys_u64(p) >= target) return;
    const unsigned wait_ms = *(volatile unsigned*)(err + 1);
    const unsigned long long limit = wait_ms ? (unsigned long long)wait_ms * 1000000ull : kPeerWaitNs;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys_u64(p) < target) {
        __nanosleep(500);
        if (globaltimer_ns() - t0 > limit) {
            atomicOr(err, kPeerErrTimeout);
            return;
        }
    }
}

// Called by every thread of every CTA after its last peer store.  Returns
// true in thread 0 of the last CTA to get here (whose later signal then
// happens after every CTA's stores); the completion counter is re-armed.
__device__ __forceinline__ bool peer_last_cta(unsigned* done) {
    __shared__ unsigned s_last;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(done, 1u);
        s_last = (prev == gridDim.x - 1) ? 1u : 0u;
        if (s_last) {
            *done = 0u;
            __threadfence_system();
        }
    }
    return threadIdx.x == 0 && s_last;
}

}  // namespace bs
