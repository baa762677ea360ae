// peer.cu — fused peer-memory routing for the PARTITIONED multi-GPU lookup
// (BASELINE.json config 5; not in the paper).  The NCCL path
// (dist.cu) stages queries into per-destination runs, exchanges counts with a
// host sync, runs two grouped Send/Recv all-to-alls and un-routes through a
// permutation.  Here the exchange is fused into the kernels that produce and
// consume it, over CUDA-IPC-mapped peer memory (NVLink / NVSwitch P2P):
//
//   k_peer_route   shard = first s with shard_max[s] >= q (else P-1); per
//                  4096-query tile, one system-scope atomicAdd per shard on
//                  rank s's receive cursor claims a slot range; the query and
//                  its 4-B tag (me << shift | i) are stored straight into rank s's
//                  receive window.  The last CTA bumps every rank's route
//                  counter.
//   k_kary_g1      (kary_g1.cuh, peer prologue/epilogue) waits for its route
//                  counter to reach t*P, looks up the *cursor received slots,
//                  and stores each GLOBAL result (base + local lb, miss bit
//                  kept) straight into the source rank's return window at the
//                  source index.  The last CTA re-arms the cursor and bumps
//                  every rank's return counter.
//   (BUCKET)       with layout.reorder = BS_REORDER_BUCKET, k_peer_wait holds
//                  the stream for the route counter and the part.cu pipeline
//                  (hist / scan / part / search / unpart) runs over the window,
//                  its size read from the cursor on the device; the unpartition
//                  stores each result into the source's return window and its
//                  last CTA re-arms the cursor and signals, as above.
//   k_peer_finish  waits for its return counter to reach t*P, copies the
//                  return window to the caller's out (or leaves the results
//                  in the window: out_local == NULL, bs_peer_results).
//
// No host synchronisation and no NCCL on the lookup path; queries and
// results cross the fabric exactly once each, with no staging copies.  The
// monotonic counters make consecutive calls safe without resets (see
// DESIGN.md §8 for the ordering argument); waits are bounded (peer_sync.cuh).
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "index.h"
#include "peer_sync.cuh"

namespace bs {

constexpr int kPeerMaxRanks = 64;
constexpr uint32_t kPeerMagic = 0x52505342u;   // "BSPR"
constexpr uint32_t kPeerVersion = 2;   // 2: 4-byte return tags

// what every rank sees of rank r (pointers valid in THIS process)
struct PeerDev {
    unsigned long long* route_sig;   // rank r's route counter
    unsigned long long* ret_sig;     // rank r's return counter
    unsigned long long* cursor;      // rank r's receive cursor
    void* win_q;                     // rank r's receive window: keys
    uint32_t* win_tag;               // rank r's receive window: (src_rank << shift) | src_idx
    uint64_t* ret;                   // rank r's return window (max_m results)
};

// control block at the start of each rank's region
struct PeerCtl {
    unsigned long long route_sig, ret_sig, cursor;
    unsigned int done_route, done_look, err;
    unsigned int wait_ms;   // bounded-wait limit, read next to err by peer_wait_ge (peer_sync.cuh)
};

struct PeerBlob {
    uint32_t magic, version, rank, world, kb, ob;
    uint64_t n_local, a_first, a_last, cap, max_m, region_bytes;
    int32_t device;
    uint32_t pad;
    cudaIpcMemHandle_t handle;
};
static_assert(sizeof(PeerBlob) <= BS_PEER_BLOB_BYTES, "peer blob too large");

struct RegionLayout {
    uint64_t q, tag, ret, total;
};

// 4-byte return tags: the source rank in the top ceil(log2 P) bits, the
// source index below (so every rank's max_m_local must be <= 2^shift)
static uint32_t tag_shift(uint32_t P) {
    uint32_t b = 0;
    while ((1u << b) < P) ++b;
    return 32 - b;
}

static uint64_t align256(uint64_t x) { return (x + 255) & ~255ull; }

static RegionLayout region_layout(uint64_t cap, uint64_t max_m, uint32_t kb) {
    RegionLayout L;
    L.q = 256;
    L.tag = align256(L.q + cap * kb);
    L.ret = align256(L.tag + cap * 4);
    L.total = align256(L.ret + (max_m ? max_m : 1) * 8);
    return L;
}

struct PeerState {
    int P = 1, rank = 0;
    uint32_t kb = 8;
    uint64_t max_m = 0, cap = 0;
    char* region = nullptr;
    RegionLayout lay{};
    cudaIpcMemHandle_t handle{};
    bool connected = false;
    uint64_t epoch = 0;
    std::vector<uint64_t> base;
    std::vector<void*> opened;       // IPC-mapped peer regions (nullptr for self)
    PeerDev* d_peers = nullptr;      // [P]
    uint64_t** d_ret = nullptr;      // [P]
    unsigned long long** d_sig = nullptr;   // [P] return counters
    uint64_t* d_shard_max = nullptr; // [P] (u64 storage, low kb bytes)
    bool bucket = false;             // lookup = the BUCKET pipeline over the window (layout.reorder)
    void* bk_ws = nullptr;           // its workspace, sized for the window (cap queries)
    uint64_t bk_ws_bytes = 0;
    PeerCtl* ctl() const { return (PeerCtl*)region; }
};

void destroy_peer_state(Index* ix) {
    PeerState* d = ix->peer;
    if (!d) return;
    for (void* p : d->opened)
        if (p) cudaIpcCloseMemHandle(p);
    void* bufs[] = {d->region, d->d_peers, d->d_ret, d->d_sig, d->d_shard_max, d->bk_ws};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete d;
    ix->peer = nullptr;
}

// One CTA routes a chunk of kRouteTile consecutive queries at a time: shard
// per query, warp-aggregated shared-memory counts give each query its rank
// within (chunk, shard), ONE system-scope atomicAdd per (chunk, shard) on the
// owner's cursor claims a contiguous slot range, then the keys and tags go
// straight into the owner's window (consecutive lanes -> consecutive slots).
constexpr int kRouteThreads = 256;
constexpr int kRoutePer = 16;
constexpr uint64_t kRouteTile = (uint64_t)kRouteThreads * kRoutePer;

template <class K>
__global__ void __launch_bounds__(kRouteThreads) k_peer_route(const K* __restrict__ q, uint64_t m,
                                                              const PeerDev* __restrict__ peers,
                                                              const uint64_t* __restrict__ shard_max, uint32_t P,
                                                              uint32_t me, uint32_t shift, uint64_t cap, unsigned* done,
                                                              unsigned* err) {
    __shared__ K s_max[kPeerMaxRanks];
    __shared__ PeerDev s_peer[kPeerMaxRanks];
    __shared__ unsigned s_cnt[kPeerMaxRanks];
    __shared__ unsigned long long s_base[kPeerMaxRanks];
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        s_max[i] = (K)shard_max[i];
        s_peer[i] = peers[i];
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t tiles = (m + kRouteTile - 1) / kRouteTile;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        const uint64_t i0 = t * kRouteTile + threadIdx.x;
        K key[kRoutePer];
        uint32_t dst[kRoutePer], rnk[kRoutePer];
#pragma unroll
        for (int j = 0; j < kRoutePer; ++j) {
            const uint64_t i = i0 + (uint64_t)j * kRouteThreads;
            const bool valid = i < m;
            key[j] = valid ? q[i] : (K)0;
            // first shard whose maximum is >= key, else the last (keeps
            // first-occurrence semantics when duplicates straddle a boundary)
            uint32_t lo = 0, hi = P - 1;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_max[mid] < key[j]) lo = mid + 1;
                else hi = mid;
            }
            dst[j] = valid ? lo : 0xFFFFFFFFu;
            const unsigned grp = __match_any_sync(0xFFFFFFFFu, dst[j]);
            const int leader = __ffs(grp) - 1;
            unsigned b = 0;
            if (valid && (int)lane == leader) b = atomicAdd(&s_cnt[lo], (unsigned)__popc(grp));
            b = __shfl_sync(0xFFFFFFFFu, b, leader);
            rnk[j] = b + __popc(grp & ((1u << lane) - 1u));
        }
        __syncthreads();
        for (uint32_t s = threadIdx.x; s < P; s += blockDim.x)
            s_base[s] = s_cnt[s] ? atomicAdd_system(s_peer[s].cursor, (unsigned long long)s_cnt[s]) : 0ull;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kRoutePer; ++j) {
            if (dst[j] == 0xFFFFFFFFu) continue;
            const uint64_t slot = s_base[dst[j]] + rnk[j];
            if (slot < cap) {
                ((K*)s_peer[dst[j]].win_q)[slot] = key[j];
                s_peer[dst[j]].win_tag[slot] = (uint32_t)(((uint64_t)me << shift) | (i0 + (uint64_t)j * kRouteThreads));
            } else {
                atomicOr(err, kPeerErrOverflow);
            }
        }
        __syncthreads();
    }
    if (peer_last_cta(done))
        for (uint32_t r = 0; r < P; ++r) red_release_sys_add_u64(s_peer[r].route_sig, 1ull);
}

constexpr int kFinishUnroll = 4;

// BUCKET lookup: the partition passes read the window with plain streaming
// loads, so they must start after every rank's route has landed — this
// one-thread kernel holds the stream until the route counter reaches target
// (the same bounded acquire the K-ary kernel does in its prologue).
__global__ void k_peer_wait(const unsigned long long* sig, unsigned long long target, unsigned* err) {
    peer_wait_ge(sig, target, err);
}

__global__ void __launch_bounds__(256) k_peer_finish(const uint64_t* ret, uint64_t m, uint64_t* __restrict__ out,
                                                     const unsigned long long* ret_sig, unsigned long long target,
                                                     unsigned* err) {
    if (threadIdx.x == 0) peer_wait_ge(ret_sig, target, err);
    __syncthreads();
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (((uintptr_t)out & 15) == 0) {
        // 16-B accesses, kFinishUnroll independent loads in flight per thread: a
        // plain 8-B grid-stride copy is latency-bound (too few bytes in flight)
        const ulonglong2* r2 = (const ulonglong2*)ret;   // the window is 256-B aligned
        ulonglong2* o2 = (ulonglong2*)out;
        const uint64_t m2 = m >> 1;
        uint64_t i = tid;
        for (; i + (kFinishUnroll - 1) * stride < m2; i += kFinishUnroll * stride) {
            ulonglong2 v[kFinishUnroll];
#pragma unroll
            for (int u = 0; u < kFinishUnroll; ++u) v[u] = __ldcg(r2 + i + u * stride);
#pragma unroll
            for (int u = 0; u < kFinishUnroll; ++u) __stcs(o2 + i + u * stride, v[u]);
        }
        for (; i < m2; i += stride) __stcs(o2 + i, __ldcg(r2 + i));
        if (tid == 0 && (m & 1)) out[m - 1] = __ldcg(ret + m - 1);
    } else {
        for (uint64_t i = tid; i < m; i += stride) out[i] = __ldcg(ret + i);
    }
}

static unsigned grid_for(uint64_t work, unsigned cap_ctas) {
    uint64_t g = (work + 255) / 256;
    if (g > cap_ctas) g = cap_ctas;
    return g ? (unsigned)g : 1u;
}

}  // namespace bs

using namespace bs;

extern "C" {

int bs_build_peer(const void* local_keys, uint64_t n_local, const bs_layout* layout, int rank, int world,
                  uint64_t max_m_local, uint64_t recv_capacity, void** out_idx) {
    if (!out_idx) return fail(BS_ERR_INVALID, "bs_build_peer: out_idx is NULL");
    *out_idx = nullptr;
    if (world < 1 || world > kPeerMaxRanks || rank < 0 || rank >= world)
        return fail(BS_ERR_INVALID, "bs_build_peer: need 0 <= rank < world <= %d", kPeerMaxRanks);
    if (max_m_local >= (1ull << 32) || max_m_local > (1ull << tag_shift((uint32_t)world)))
        return fail(BS_ERR_INVALID, "bs_build_peer: max_m_local must be < 2^32 and <= 2^(32 - ceil(log2 world)) (4-B tags)");
    int rc = bs_build(local_keys, n_local, layout, out_idx);
    if (rc != BS_OK) return rc;
    Index* ix = (Index*)*out_idx;
    auto cleanup = [&](int code) { bs_destroy(ix); *out_idx = nullptr; return code; };
    if (ix->ob != 8) return cleanup(fail(BS_ERR_INVALID, "bs_build_peer: needs out_bytes = 8 (global ranks)"));
    if (ix->layout.variant != BS_VARIANT_KARY)
        return cleanup(fail(BS_ERR_UNSUPPORTED, "bs_build_peer: needs variant KARY (the g1 kernel carries the peer epilogue)"));
    // reject, after the AUTO choices are resolved, every layout the g1 kernel cannot
    // run: a lookup would otherwise fail only after its route kernel had already
    // filled the peers' windows and bumped their counters
    const bool bucket = ix->layout.reorder == BS_REORDER_BUCKET;
    if (!bucket && !g1_shape_ok(ix))
        return cleanup(fail(BS_ERR_UNSUPPORTED, "bs_build_peer: layout needs kary_mode 6/7 with W*key <= 64 B and "
                                                "C*key in 32..256 B (got mode %u, W %u, C %u, key %u B)",
                            ix->layout.kary_mode, ix->kW, ix->kC, ix->kb));
    PeerState* d = new PeerState();
    ix->peer = d;
    d->P = world;
    d->rank = rank;
    d->kb = ix->kb;
    d->max_m = max_m_local;
    d->cap = recv_capacity ? recv_capacity : (uint64_t)world * (max_m_local ? max_m_local : 1);
    if (d->cap >= (1ull << 40)) return cleanup(fail(BS_ERR_INVALID, "bs_build_peer: recv_capacity too large"));
    if (bucket) {
        // the window is partitioned in place of a caller batch: workspace for cap queries
        if (!ix->bk.mx || !bucket_workspace_bytes(ix->bk.B, d->cap, ix->kb, 8, (uint32_t)ix->sm_count, &d->bk_ws_bytes))
            return cleanup(fail(BS_ERR_UNSUPPORTED, "bs_build_peer: BS_REORDER_BUCKET needs n_local <= %llu keys and "
                                                    "recv_capacity < 2^32",
                                (unsigned long long)bucket_max_keys(ix->kb)));
        cudaError_t e = cudaMalloc(&d->bk_ws, d->bk_ws_bytes);
        if (e != cudaSuccess) return cleanup(fail(BS_ERR_OOM, "bs_build_peer: cudaMalloc(%llu B bucket workspace): %s",
                                                  (unsigned long long)d->bk_ws_bytes, cudaGetErrorString(e)));
        d->bucket = true;
    }
    d->lay = region_layout(d->cap, d->max_m, d->kb);
    cudaError_t e = cudaMalloc(&d->region, d->lay.total);
    if (e != cudaSuccess) return cleanup(fail(BS_ERR_OOM, "bs_build_peer: cudaMalloc(%llu B window): %s",
                                              (unsigned long long)d->lay.total, cudaGetErrorString(e)));
    e = cudaMemset(d->region, 0, 256);
    if (e == cudaSuccess) {
        // bounded waits: BS_PEER_WAIT_MS (default 20000) before a wait gives up
        unsigned wait_ms = 20000;
        if (const char* v = getenv("BS_PEER_WAIT_MS")) {
            const long x = atol(v);
            if (x > 0 && x < 3600000) wait_ms = (unsigned)x;
        }
        e = cudaMemcpy((char*)d->region + offsetof(PeerCtl, wait_ms), &wait_ms, sizeof wait_ms, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&d->handle, d->region);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_peers, sizeof(PeerDev) * world);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_ret, sizeof(uint64_t*) * world);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_sig, sizeof(unsigned long long*) * world);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_shard_max, sizeof(uint64_t) * world);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cleanup(fail_cuda(e, "bs_build_peer: window setup"));
    return BS_OK;
}

int bs_peer_export(const void* idx, void* blob) {
    if (!idx || !blob) return fail(BS_ERR_INVALID, "bs_peer_export: NULL");
    const Index* ix = (const Index*)idx;
    const PeerState* d = ix->peer;
    if (!d) return fail(BS_ERR_INVALID, "bs_peer_export: index was not built with bs_build_peer");
    PeerBlob b;
    memset(&b, 0, sizeof b);
    b.magic = kPeerMagic;
    b.version = kPeerVersion;
    b.rank = (uint32_t)d->rank;
    b.world = (uint32_t)d->P;
    b.kb = ix->kb;
    b.ob = ix->ob;
    b.n_local = ix->n;
    b.a_first = ix->a_first;
    b.a_last = ix->a_last;
    b.cap = d->cap;
    b.max_m = d->max_m;
    b.region_bytes = d->lay.total;
    b.device = ix->device;
    b.handle = d->handle;
    memset(blob, 0, BS_PEER_BLOB_BYTES);
    memcpy(blob, &b, sizeof b);
    return BS_OK;
}

int bs_peer_connect(void* idx, const void* blobs) {
    if (!idx || !blobs) return fail(BS_ERR_INVALID, "bs_peer_connect: NULL");
    Index* ix = (Index*)idx;
    PeerState* d = ix->peer;
    if (!d) return fail(BS_ERR_INVALID, "bs_peer_connect: index was not built with bs_build_peer");
    if (d->connected) return fail(BS_ERR_INVALID, "bs_peer_connect: already connected");
    const int P = d->P;
    std::vector<PeerBlob> B(P);
    for (int r = 0; r < P; ++r) {
        memcpy(&B[r], (const char*)blobs + (size_t)r * BS_PEER_BLOB_BYTES, sizeof(PeerBlob));
        const PeerBlob& b = B[r];
        if (b.magic != kPeerMagic || b.version != kPeerVersion)
            return fail(BS_ERR_INVALID, "bs_peer_connect: blob %d is not a bs_peer_export blob", r);
        if ((int)b.rank != r || (int)b.world != P || b.kb != ix->kb || b.ob != 8)
            return fail(BS_ERR_INVALID, "bs_peer_connect: blob %d has rank %u world %u kb %u (expected %d/%d/%u)", r,
                        b.rank, b.world, b.kb, r, P, ix->kb);
    }
    // shards must be globally ordered by rank; global rank of shard r = sum of earlier sizes
    d->base.assign(P, 0);
    uint64_t acc = 0;
    std::vector<uint64_t> mx(P);
    for (int r = 0; r < P; ++r) {
        d->base[r] = acc;
        acc += B[r].n_local;
        mx[r] = B[r].a_last;
        if (r + 1 < P) {
            const bool ok = ix->kb == 8 ? B[r].a_last <= B[r + 1].a_first
                                        : (uint32_t)B[r].a_last <= (uint32_t)B[r + 1].a_first;
            if (!ok) return fail(BS_ERR_NOT_SORTED, "bs_peer_connect: max of shard %d > min of shard %d", r, r + 1);
        }
    }
    d->opened.assign(P, nullptr);
    std::vector<PeerDev> pd(P);
    std::vector<uint64_t*> rp(P);
    std::vector<unsigned long long*> sp(P);
    for (int r = 0; r < P; ++r) {
        char* base = nullptr;
        if (r == d->rank) {
            base = d->region;
        } else {
            void* p = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&p, B[r].handle, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                for (void*& o : d->opened)
                    if (o) { cudaIpcCloseMemHandle(o); o = nullptr; }
                return fail_cuda(e, "bs_peer_connect: cudaIpcOpenMemHandle");
            }
            d->opened[r] = p;
            base = (char*)p;
        }
        const RegionLayout L = region_layout(B[r].cap, B[r].max_m, ix->kb);
        PeerCtl* c = (PeerCtl*)base;
        pd[r] = PeerDev{&c->route_sig, &c->ret_sig, &c->cursor, base + L.q, (uint32_t*)(base + L.tag),
                        (uint64_t*)(base + L.ret)};
        rp[r] = pd[r].ret;
        sp[r] = pd[r].ret_sig;
    }
    cudaError_t e = cudaMemcpy(d->d_peers, pd.data(), sizeof(PeerDev) * P, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d->d_ret, rp.data(), sizeof(uint64_t*) * P, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d->d_sig, sp.data(), sizeof(unsigned long long*) * P, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d->d_shard_max, mx.data(), sizeof(uint64_t) * P, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail_cuda(e, "bs_peer_connect: peer tables");
    d->connected = true;
    return BS_OK;
}

int bs_lookup_peer(const void* idx, const void* local_queries, uint64_t m_local, void* out_local, void* stream) {
    if (!idx) return fail(BS_ERR_INVALID, "bs_lookup_peer: idx is NULL");
    const Index* ix = (const Index*)idx;
    PeerState* d = ix->peer;
    if (!d || !d->connected) return fail(BS_ERR_INVALID, "bs_lookup_peer: index not built with bs_build_peer / not connected");
    if (m_local > d->max_m) return fail(BS_ERR_INVALID, "bs_lookup_peer: m_local > max_m_local given at build");
    if (m_local && !local_queries) return fail(BS_ERR_INVALID, "bs_lookup_peer: NULL queries");
    if ((uintptr_t)local_queries % ix->kb || (uintptr_t)out_local % 8)
        return fail(BS_ERR_INVALID, "bs_lookup_peer: misaligned queries/out");
    if (!d->bucket && !g1_shape_ok(ix)) return fail(BS_ERR_UNSUPPORTED, "bs_lookup_peer: layout cannot run the g1 kernel");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t P = (uint32_t)d->P, me = (uint32_t)d->rank;
    PeerCtl* c = d->ctl();
    const unsigned long long target = (unsigned long long)(d->epoch + 1) * P;
    uint64_t tiles = (m_local + kRouteTile - 1) / kRouteTile;
    const unsigned gr = (unsigned)(tiles < 1 ? 1 : tiles > (uint64_t)ix->sm_count * 8 ? (uint64_t)ix->sm_count * 8 : tiles);
    if (ix->kb == 8)
        k_peer_route<uint64_t><<<gr, 256, 0, s>>>((const uint64_t*)local_queries, m_local, d->d_peers, d->d_shard_max, P,
                                                  me, tag_shift(P), d->cap, &c->done_route, &c->err);
    else
        k_peer_route<uint32_t><<<gr, 256, 0, s>>>((const uint32_t*)local_queries, m_local, d->d_peers, d->d_shard_max, P,
                                                  me, tag_shift(P), d->cap, &c->done_route, &c->err);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "k_peer_route launch");
    bs_launch L;
    bs_launch_default(idx, &L);
    PeerLaunch pl{&c->cursor, &c->route_sig, target, (const uint32_t*)(d->region + d->lay.tag), d->d_ret, d->d_sig,
                  &c->done_look, &c->err, d->base[me], P, tag_shift(P)};
    // once the route kernel is queued the call is committed: every rank waits
    // for this one, so a failure past this point is fatal for the group
    d->epoch += 1;
    if (d->bucket) {
        // route -> wait -> hist / scan / part / search / unpart over the window;
        // the unpartition stores each result into its source's return window
        k_peer_wait<<<1, 1, 0, s>>>(&c->route_sig, target, &c->err);
        count_launch();
        BucketPeer bp;
        bp.m_dev = &c->cursor;
        bp.m_hint = d->max_m;
        bp.tag = (const uint32_t*)(d->region + d->lay.tag);
        bp.ret = d->d_ret;
        bp.sig = d->d_sig;
        bp.cursor = &c->cursor;
        bp.done = &c->done_look;
        bp.base = d->base[me];
        bp.P = P;
        bp.shift = tag_shift(P);
        bool uns = false;
        uint32_t chunk = 0;
        if (const char* v = getenv("BS_BUCKET_CHUNK")) chunk = (uint32_t)atoi(v);
        e = launch_bucket(ix->kb, 8, ix->bk, ix->d_keys, ix->n, d->region + d->lay.q, d->cap, nullptr,
                          (L.cache_hints & BS_HINT_STREAM_EVICT_FIRST) ? 1u : 0u, chunk, d->bk_ws, d->bk_ws_bytes,
                          (uint32_t)ix->sm_count, s, &uns, 0, nullptr, &bp);
        if (uns) return fail(BS_ERR_UNSUPPORTED, "bs_lookup_peer: bucket pipeline cannot run this window");
        if (e != cudaSuccess) return fail_cuda(e, "bs_lookup_peer: bucket pipeline launch");
    } else {
        int rc = dispatch_kary_peer(ix, d->region + d->lay.q, d->cap, s, L, pl);
        if (rc != BS_OK) return rc;
    }
    // out_local == NULL: the results stay in the return window (bs_peer_results)
    const uint64_t mc = out_local ? m_local : 0;
    k_peer_finish<<<grid_for(mc / 2, (unsigned)ix->sm_count * 8), 256, 0, s>>>(
        (const uint64_t*)(d->region + d->lay.ret), mc, (uint64_t*)out_local, &c->ret_sig, target, &c->err);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "k_peer_finish launch");
    return BS_OK;
}

int bs_peer_results(const void* idx, const void** results) {
    if (!idx || !results) return fail(BS_ERR_INVALID, "bs_peer_results: NULL");
    const PeerState* d = ((const Index*)idx)->peer;
    if (!d) return fail(BS_ERR_INVALID, "bs_peer_results: index was not built with bs_build_peer");
    *results = d->region + d->lay.ret;
    return BS_OK;
}

int bs_peer_status(const void* idx, uint32_t* err_bits, uint64_t* calls) {
    if (!idx || !err_bits) return fail(BS_ERR_INVALID, "bs_peer_status: NULL");
    const Index* ix = (const Index*)idx;
    const PeerState* d = ix->peer;
    if (!d) return fail(BS_ERR_INVALID, "bs_peer_status: index was not built with bs_build_peer");
    PeerCtl c;
    cudaError_t e = cudaMemcpy(&c, d->region, sizeof c, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail_cuda(e, "bs_peer_status");
    *err_bits = c.err;
    if (calls) *calls = d->epoch;
    return BS_OK;
}

}  // extern "C"
