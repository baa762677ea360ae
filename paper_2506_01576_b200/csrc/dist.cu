// dist.cu — multi-GPU entry points (BASELINE.json configs 4-5; not in the paper).
//
// One process per GPU.  REPLICATED: each rank holds the whole index, the
// caller shards queries, no collective on the lookup path.  PARTITIONED: rank
// r holds the contiguous rank range [base_r, base_r + n_r) of the global
// sorted array; a lookup is
//   k_route_count  (shard = first s with shard_max[s] >= q, else P-1; per-shard counts)
//   ncclAllGather  (P x P count matrix; one host sync to size the exchange)
//   k_route_scatter (queries grouped by destination, permutation kept)
//   grouped ncclSend/ncclRecv of the queries (NVLink / NVSwitch)
//   local lookup (the index's variant) + k_add_base (global rank, miss bit kept)
//   grouped ncclSend/ncclRecv of the results back
//   k_unroute      (results back into the caller's query order)
// Routing by shard maxima keeps first-occurrence semantics when a run of
// duplicates straddles a shard boundary (tests/test_dist_cpu.py).
#include <cstring>
#include <vector>

#include "index.h"

#ifdef BS_HAVE_NCCL
#include <nccl.h>
#endif

namespace bs {

constexpr int kMaxShards = 64;

#ifdef BS_HAVE_NCCL
struct DistComm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
};
#endif

struct DistState {
    int mode = BS_DIST_REPLICATED;
#ifdef BS_HAVE_NCCL
    DistComm* comm = nullptr;
#endif
    int P = 1, rank = 0;
    uint64_t max_m = 0;
    uint64_t recv_cap = 0;            // sum of every rank's max_m_local (receive buffer slots)
    std::vector<uint64_t> base;       // global rank of each shard's first key
    void* d_shard_max = nullptr;      // P keys (u64 storage)
    uint8_t* d_dest = nullptr;        // per query destination
    uint32_t* d_perm = nullptr;       // per query slot in the send buffer
    uint64_t* d_counts = nullptr;     // P (mine) + P*P (gathered) + P cursors
    void* d_sendq = nullptr;          // max_m keys
    void* d_recvq = nullptr;          // recv_cap keys
    uint64_t* d_recvres = nullptr;    // recv_cap results
    uint64_t* d_backres = nullptr;    // max_m results
    void* d_ws = nullptr;             // workspace of the owner's out-of-place lookup (layout.reorder
    uint64_t ws_bytes = 0;            // GLOBAL / BUCKET) for recv_cap queries; NULL: in-place lookup
};

void destroy_dist_state(Index* ix) {
    DistState* d = ix->dist;
    if (!d) return;
    void* bufs[] = {d->d_shard_max, d->d_dest, d->d_perm, d->d_counts, d->d_sendq, d->d_recvq, d->d_recvres,
                    d->d_backres, d->d_ws};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete d;
    ix->dist = nullptr;
}

template <class K>
__global__ void k_route_count(const K* __restrict__ q, uint64_t m, const K* __restrict__ smax, int P,
                              uint8_t* __restrict__ dest, unsigned long long* __restrict__ counts) {
    __shared__ K s_max[kMaxShards];
    __shared__ unsigned int s_cnt[kMaxShards];
    for (int i = threadIdx.x; i < P; i += blockDim.x) { s_max[i] = smax[i]; s_cnt[i] = 0; }
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const K key = q[i];
        int s = 0;
        while (s < P - 1 && s_max[s] < key) ++s;   // first shard whose max >= q, else the last
        dest[i] = (uint8_t)s;
        atomicAdd(&s_cnt[s], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(&counts[i], (unsigned long long)s_cnt[i]);
}

// Per tile of 4096 queries: warp-aggregated shared-memory ranks per
// destination, ONE global atomicAdd per (tile, destination) on its cursor,
// then the queries go to consecutive slots of their destination's run
// (consecutive lanes -> consecutive slots).  A per-warp global atomic on the
// P cursors (the first version) serialised ~4 M atomics on one address at
// world 1: 4.0 ms vs 0.5 ms for this form (profiles/r1s3j_*).
constexpr int kScatterThreads = 256;
constexpr int kScatterPer = 16;
constexpr uint64_t kScatterTile = (uint64_t)kScatterThreads * kScatterPer;

template <class K>
__global__ void __launch_bounds__(kScatterThreads) k_route_scatter(const K* __restrict__ q, uint64_t m,
                                                                   const uint8_t* __restrict__ dest,
                                                                   const unsigned long long* __restrict__ offs,
                                                                   unsigned long long* __restrict__ cursor,
                                                                   K* __restrict__ sendq, uint32_t* __restrict__ perm,
                                                                   int P) {
    __shared__ unsigned s_cnt[kMaxShards];
    __shared__ unsigned long long s_base[kMaxShards];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t tiles = (m + kScatterTile - 1) / kScatterTile;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        const uint64_t i0 = t * kScatterTile + threadIdx.x;
        uint32_t dst[kScatterPer], rnk[kScatterPer];
#pragma unroll
        for (int j = 0; j < kScatterPer; ++j) {
            const uint64_t i = i0 + (uint64_t)j * kScatterThreads;
            dst[j] = i < m ? (uint32_t)dest[i] : 0xFFFFFFFFu;
            const unsigned grp = __match_any_sync(0xFFFFFFFFu, dst[j]);
            const int leader = __ffs(grp) - 1;
            unsigned b = 0;
            if (dst[j] != 0xFFFFFFFFu && (int)lane == leader) b = atomicAdd(&s_cnt[dst[j]], (unsigned)__popc(grp));
            b = __shfl_sync(0xFFFFFFFFu, b, leader);
            rnk[j] = b + __popc(grp & ((1u << lane) - 1u));
        }
        __syncthreads();
        for (int s = threadIdx.x; s < P; s += blockDim.x)
            s_base[s] = s_cnt[s] ? offs[s] + atomicAdd(&cursor[s], (unsigned long long)s_cnt[s]) : 0ull;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kScatterPer; ++j) {
            if (dst[j] == 0xFFFFFFFFu) continue;
            const uint64_t i = i0 + (uint64_t)j * kScatterThreads;
            const uint64_t pos = s_base[dst[j]] + rnk[j];
            sendq[pos] = q[i];
            perm[i] = (uint32_t)pos;
        }
        __syncthreads();
    }
}

__global__ void k_add_base(uint64_t* __restrict__ res, uint64_t cnt, uint64_t base) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = res[i];
        const uint64_t miss = r & (1ull << 63);
        res[i] = ((r & ~(1ull << 63)) + base) | miss;
    }
}

__global__ void k_unroute(const uint64_t* __restrict__ back, const uint32_t* __restrict__ perm, uint64_t m,
                          uint64_t* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = back[perm[i]];
}

static unsigned grid_of(uint64_t work) {
    uint64_t g = (work + 255) / 256;
    if (g > 148ull * 16) g = 148ull * 16;
    return g ? (unsigned)g : 1u;
}

}  // namespace bs

using namespace bs;

extern "C" {

#ifdef BS_HAVE_NCCL

static int nccl_fail(ncclResult_t r, const char* what) {
    return fail(BS_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

int bs_dist_get_uid(void* uid) {
    if (!uid) return fail(BS_ERR_INVALID, "bs_dist_get_uid: NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(uid, &id, sizeof id);
    return BS_OK;
}

int bs_dist_init(const void* uid, int rank, int world, void** out_comm) {
    if (!uid || !out_comm || world < 1 || rank < 0 || rank >= world || world > kMaxShards)
        return fail(BS_ERR_INVALID, "bs_dist_init: bad arguments (world must be 1..%d)", kMaxShards);
    ncclUniqueId id;
    memcpy(&id, uid, sizeof id);
    DistComm* c = new DistComm();
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) { delete c; return nccl_fail(r, "ncclCommInitRank"); }
    c->rank = rank;
    c->world = world;
    *out_comm = c;
    return BS_OK;
}

void bs_dist_destroy(void* comm) {
    DistComm* c = (DistComm*)comm;
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

int bs_build_dist(void* comm, const void* local_keys, uint64_t n_local, int mode, const bs_layout* layout,
                  uint64_t max_m_local, void** out_idx) {
    if (!comm || !out_idx) return fail(BS_ERR_INVALID, "bs_build_dist: NULL");
    if (mode != BS_DIST_REPLICATED && mode != BS_DIST_PARTITIONED) return fail(BS_ERR_INVALID, "bs_build_dist: bad mode");
    if (max_m_local >= (1ull << 32)) return fail(BS_ERR_INVALID, "bs_build_dist: max_m_local must be < 2^32");
    DistComm* c = (DistComm*)comm;
    int rc = bs_build(local_keys, n_local, layout, out_idx);
    if (rc != BS_OK) return rc;
    Index* ix = (Index*)*out_idx;
    DistState* d = new DistState();
    ix->dist = d;
    d->comm = c;
    d->mode = mode;
    d->P = c->world;
    d->rank = c->rank;
    d->max_m = max_m_local;
    if (mode == BS_DIST_REPLICATED) return BS_OK;
    if (ix->ob != 8) { bs_destroy(ix); *out_idx = nullptr; return fail(BS_ERR_INVALID, "PARTITIONED needs out_bytes = 8"); }

    const int P = d->P;
    const uint32_t kb = ix->kb;
    cudaError_t e;
    auto cleanup = [&](int code) { bs_destroy(ix); *out_idx = nullptr; return code; };
    // (min, max, n, max_m_local) of every shard: every rank sizes its receive
    // buffers from the SUM of all ranks' max_m_local, so a receive can never
    // overflow and no rank ever has to leave a collective early
    constexpr int NM = 4;
    uint64_t* d_meta = nullptr;
    e = cudaMalloc(&d_meta, sizeof(uint64_t) * NM * (P + 1));
    if (e != cudaSuccess) return cleanup(fail_cuda(e, "cudaMalloc(meta)"));
    uint64_t mine[NM] = {ix->a_first, ix->a_last, n_local, max_m_local};
    cudaMemcpy(d_meta, mine, sizeof mine, cudaMemcpyHostToDevice);
    ncclResult_t r = ncclAllGather(d_meta, d_meta + NM, NM, ncclUint64, c->comm, 0);
    if (r != ncclSuccess) { cudaFree(d_meta); return cleanup(nccl_fail(r, "ncclAllGather(meta)")); }
    std::vector<uint64_t> meta(NM * P);
    e = cudaMemcpy(meta.data(), d_meta + NM, sizeof(uint64_t) * NM * P, cudaMemcpyDeviceToHost);
    cudaFree(d_meta);
    if (e != cudaSuccess) return cleanup(fail_cuda(e, "meta copy"));
    d->base.assign(P, 0);
    uint64_t acc = 0;
    d->recv_cap = 0;
    for (int s = 0; s < P; ++s) {
        d->base[s] = acc;
        acc += meta[NM * s + 2];
        d->recv_cap += meta[NM * s + 3];
        if (s + 1 < P) {
            const uint64_t mx = meta[NM * s + 1], mn_next = meta[NM * (s + 1)];
            const bool ok = kb == 8 ? mx <= mn_next : (uint32_t)mx <= (uint32_t)mn_next;
            if (!ok) return cleanup(fail(BS_ERR_NOT_SORTED, "PARTITIONED: max of shard %d > min of shard %d", s, s + 1));
        }
    }
    // shard maxima in the key width, on the device
    e = cudaMalloc(&d->d_shard_max, 8 * P);
    if (e != cudaSuccess) return cleanup(fail_cuda(e, "cudaMalloc(shard_max)"));
    std::vector<uint64_t> mx64(P);
    std::vector<uint32_t> mx32(P);
    for (int s = 0; s < P; ++s) { mx64[s] = meta[NM * s + 1]; mx32[s] = (uint32_t)meta[NM * s + 1]; }
    cudaMemcpy(d->d_shard_max, kb == 8 ? (void*)mx64.data() : (void*)mx32.data(), kb * P, cudaMemcpyHostToDevice);
    const uint64_t M = max_m_local ? max_m_local : 1;
    const uint64_t R = d->recv_cap ? d->recv_cap : 1;
    struct { void** p; size_t b; } allocs[] = {
        {(void**)&d->d_dest, M}, {(void**)&d->d_perm, 4 * M}, {(void**)&d->d_counts, 8 * (size_t)(P * P + 3 * P)},
        {&d->d_sendq, kb * M}, {&d->d_recvq, kb * R}, {(void**)&d->d_recvres, 8 * R},
        {(void**)&d->d_backres, 8 * M}};
    for (auto& a : allocs) {
        e = cudaMalloc(a.p, a.b);
        if (e != cudaSuccess) return cleanup(fail_cuda(e, "cudaMalloc(exchange buffers)"));
    }
    // the owner's lookup of the received queries in the layout's out-of-place
    // mode (the same local lookup as the fused peer path): its workspace, sized
    // for the receive capacity; a layout / size the mode cannot take keeps the
    // in-place lookup
    const uint32_t ro = ix->layout.reorder;
    if (ro == BS_REORDER_GLOBAL || ro == BS_REORDER_BUCKET) {
        uint64_t wb = 0;
        if (bs_workspace_bytes(ix, R, nullptr, &wb) == BS_OK && wb) {
            e = cudaMalloc(&d->d_ws, wb);
            if (e != cudaSuccess) return cleanup(fail(BS_ERR_OOM, "bs_build_dist: cudaMalloc(%llu B lookup workspace)",
                                                      (unsigned long long)wb));
            d->ws_bytes = wb;
        }
    }
    return BS_OK;
}

int bs_lookup_dist(const void* idx, const void* local_queries, uint64_t m_local, void* out_local, void* stream) {
    if (!idx) return fail(BS_ERR_INVALID, "bs_lookup_dist: idx is NULL");
    const Index* ix = (const Index*)idx;
    DistState* d = ix->dist;
    if (!d) return fail(BS_ERR_INVALID, "bs_lookup_dist: index was not built with bs_build_dist");
    if (d->mode == BS_DIST_REPLICATED) return bs_lookup(idx, local_queries, m_local, out_local, stream);
    // a bad call still takes part in every collective (with nothing to route),
    // so the other ranks never wait on a rank that left early; it fails at the end
    const char* bad = nullptr;
    if (m_local > d->max_m) bad = "bs_lookup_dist: m_local > max_m_local given at build";
    else if (m_local && (!local_queries || !out_local)) bad = "bs_lookup_dist: NULL buffers";
    if (bad) m_local = 0;
    cudaStream_t s = (cudaStream_t)stream;
    const int P = d->P, me = d->rank;
    const uint32_t kb = ix->kb;
    ncclComm_t comm = d->comm->comm;
    unsigned long long* cnt = (unsigned long long*)d->d_counts;   // [P] mine
    unsigned long long* all = cnt + P;                             // [P*P] gathered
    unsigned long long* offs = all + P * P;                        // [P] my send offsets
    unsigned long long* cur = offs + P;                            // [P] cursors
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (P * P + 3 * P), s);
    if (e != cudaSuccess) return fail_cuda(e, "dist memset");
    if (m_local) {
        if (kb == 8)
            k_route_count<uint64_t><<<grid_of(m_local), 256, 0, s>>>((const uint64_t*)local_queries, m_local,
                                                                     (const uint64_t*)d->d_shard_max, P, d->d_dest, cnt);
        else
            k_route_count<uint32_t><<<grid_of(m_local), 256, 0, s>>>((const uint32_t*)local_queries, m_local,
                                                                     (const uint32_t*)d->d_shard_max, P, d->d_dest, cnt);
        count_launch();
    }
    ncclResult_t r = ncclAllGather(cnt, all, P, ncclUint64, comm, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather(counts)");
    std::vector<unsigned long long> mat(P * P);
    e = cudaMemcpyAsync(mat.data(), all, sizeof(unsigned long long) * P * P, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail_cuda(e, "dist count exchange");
    // row r = what rank r sends to each shard
    std::vector<unsigned long long> soff(P), rcnt(P), roff(P);
    unsigned long long acc = 0, racc = 0;
    for (int t = 0; t < P; ++t) {
        soff[t] = acc;
        acc += mat[me * P + t];
        rcnt[t] = mat[t * P + me];
        roff[t] = racc;
        racc += rcnt[t];
    }
    // racc <= sum of every rank's m_local <= sum of max_m_local = recv_cap (sized at build)
    e = cudaMemcpyAsync(offs, soff.data(), sizeof(unsigned long long) * P, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return fail_cuda(e, "dist offsets");
    const uint64_t sc_tiles = (m_local + kScatterTile - 1) / kScatterTile;
    const unsigned grid_scatter = (unsigned)(sc_tiles > 148ull * 8 ? 148ull * 8 : (sc_tiles ? sc_tiles : 1));
    if (m_local) {
        if (kb == 8)
            k_route_scatter<uint64_t><<<grid_scatter, kScatterThreads, 0, s>>>((const uint64_t*)local_queries, m_local,
                                                                             d->d_dest, offs, cur, (uint64_t*)d->d_sendq,
                                                                             d->d_perm, P);
        else
            k_route_scatter<uint32_t><<<grid_scatter, kScatterThreads, 0, s>>>((const uint32_t*)local_queries, m_local,
                                                                             d->d_dest, offs, cur, (uint32_t*)d->d_sendq,
                                                                             d->d_perm, P);
        count_launch();
    }
    const ncclDataType_t kt = kb == 8 ? ncclUint64 : ncclUint32;
    ncclGroupStart();
    for (int t = 0; t < P; ++t) {
        const unsigned long long sc = mat[me * P + t];
        if (sc) ncclSend((const char*)d->d_sendq + soff[t] * kb, sc, kt, t, comm, s);
        if (rcnt[t]) ncclRecv((char*)d->d_recvq + roff[t] * kb, rcnt[t], kt, t, comm, s);
    }
    r = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "query all-to-all");
    if (racc) {
        bs_launch Ld;
        bs_launch_default(idx, &Ld);
        int rc;
        if (d->d_ws) {
            rc = bs_lookup_ws(idx, d->d_recvq, racc, d->d_recvres, s, &Ld, d->d_ws, d->ws_bytes);
        } else {
            if (Ld.reorder == BS_REORDER_GLOBAL || Ld.reorder == BS_REORDER_BUCKET) Ld.reorder = BS_REORDER_NONE;
            rc = bs_lookup_ex(idx, d->d_recvq, racc, d->d_recvres, s, &Ld);
        }
        if (rc != BS_OK) return rc;
        k_add_base<<<grid_of(racc), 256, 0, s>>>(d->d_recvres, racc, d->base[me]);
        count_launch();
    }
    ncclGroupStart();
    for (int t = 0; t < P; ++t) {
        const unsigned long long sc = mat[me * P + t];
        if (rcnt[t]) ncclSend(d->d_recvres + roff[t], rcnt[t], ncclUint64, t, comm, s);
        if (sc) ncclRecv(d->d_backres + soff[t], sc, ncclUint64, t, comm, s);
    }
    r = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "result all-to-all");
    if (m_local) {
        k_unroute<<<grid_of(m_local), 256, 0, s>>>(d->d_backres, d->d_perm, m_local, (uint64_t*)out_local);
        count_launch();
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "dist kernels");
    if (bad) return fail(BS_ERR_INVALID, "%s", bad);
    return BS_OK;
}

#else  // no NCCL headers at build time

int bs_dist_get_uid(void*) { return fail(BS_ERR_UNSUPPORTED, "libbs built without NCCL"); }
int bs_dist_init(const void*, int, int, void**) { return fail(BS_ERR_UNSUPPORTED, "libbs built without NCCL"); }
void bs_dist_destroy(void*) {}
int bs_build_dist(void*, const void*, uint64_t, int, const bs_layout*, uint64_t, void**) {
    return fail(BS_ERR_UNSUPPORTED, "libbs built without NCCL");
}
int bs_lookup_dist(const void*, const void*, uint64_t, void*, void*) {
    return fail(BS_ERR_UNSUPPORTED, "libbs built without NCCL");
}

#endif

}  // extern "C"
