// host.cu — bs_lookup_host: end-to-end lookups from host memory.
//
// Chunked S-stream pipeline (S = 4 by default): for chunk c on stream c % S:
//   H2D(queries chunk) -> bs lookup kernel -> D2H(results chunk)
// so the PCIe copy of chunk c+1 overlaps the kernel of chunk c and the
// copy-back of chunk c-1 (H2D and D2H use separate copy engines).  Pageable
// host buffers are staged through pinned buffers by the calling thread.
#include <cstdlib>
#include <cstring>

#include "index.h"

namespace bs {

constexpr int kMaxStages = 8;

struct HostCtx {
    uint64_t chunk = 0;                 // queries per chunk
    int stages = 4;                     // buffers / streams in the ring
    cudaStream_t st[kMaxStages] = {};
    cudaEvent_t done[kMaxStages] = {};
    void* dq[kMaxStages] = {};
    void* dout[kMaxStages] = {};
    void* hq[kMaxStages] = {};          // pinned staging (pageable callers only)
    void* hout[kMaxStages] = {};
};

void destroy_host_ctx(Index* ix) {
    HostCtx* h = ix->host;
    if (!h) return;
    for (int i = 0; i < kMaxStages; ++i) {
        if (h->st[i]) cudaStreamSynchronize(h->st[i]);
        if (h->dq[i]) cudaFree(h->dq[i]);
        if (h->dout[i]) cudaFree(h->dout[i]);
        if (h->hq[i]) cudaFreeHost(h->hq[i]);
        if (h->hout[i]) cudaFreeHost(h->hout[i]);
        if (h->done[i]) cudaEventDestroy(h->done[i]);
        if (h->st[i]) cudaStreamDestroy(h->st[i]);
    }
    delete h;
    ix->host = nullptr;
}

static int make_ctx(Index* ix) {
    HostCtx* h = new HostCtx();
    h->chunk = 1ull << 22;   // 4 Mi queries: 32 MB per buffer at u64
    // tuning knobs for the copy pipeline (not part of the ABI)
    if (const char* e = getenv("BS_HOST_CHUNK_LOG2")) {
        const int v = atoi(e);
        if (v >= 16 && v <= 26) h->chunk = 1ull << v;
    }
    if (const char* e = getenv("BS_HOST_STAGES")) {
        const int v = atoi(e);
        if (v >= 2 && v <= kMaxStages) h->stages = v;
    }
    ix->host = h;
    for (int i = 0; i < h->stages; ++i) {
        cudaError_t e = cudaStreamCreateWithFlags(&h->st[i], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->done[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaMalloc(&h->dq[i], h->chunk * ix->kb);
        if (e == cudaSuccess) e = cudaMalloc(&h->dout[i], h->chunk * ix->ob);
        if (e == cudaSuccess) e = cudaMallocHost(&h->hq[i], h->chunk * ix->kb);
        if (e == cudaSuccess) e = cudaMallocHost(&h->hout[i], h->chunk * ix->ob);
        if (e != cudaSuccess) {
            destroy_host_ctx(ix);
            return fail_cuda(e, "bs_lookup_host: staging allocation");
        }
    }
    return BS_OK;
}

static bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
}

}  // namespace bs

using namespace bs;

extern "C" int bs_lookup_host(const void* idx, const void* host_q, uint64_t m, void* host_out, void* stream) {
    if (!idx) return fail(BS_ERR_INVALID, "bs_lookup_host: idx is NULL");
    if (m == 0) return BS_OK;
    if (!host_q || !host_out) return fail(BS_ERR_INVALID, "bs_lookup_host: NULL buffers with m > 0");
    Index* ix = (Index*)idx;
    std::lock_guard<std::mutex> lock(ix->host_mu);
    if (!ix->host) {
        int rc = make_ctx(ix);
        if (rc != BS_OK) return rc;
    }
    HostCtx* h = ix->host;
    bs_launch L;
    bs_launch_default(idx, &L);
    // chunks are looked up in the index's default mode; the out-of-place GLOBAL /
    // BUCKET reorderings need a caller workspace, so chunks take the in-place path
    if (L.reorder == BS_REORDER_GLOBAL || L.reorder == BS_REORDER_BUCKET) L.reorder = BS_REORDER_NONE;
    const bool pin_q = is_pinned(host_q), pin_o = is_pinned(host_out);
    const uint32_t kb = ix->kb, ob = ix->ob;

    // order after prior work on the caller's stream
    cudaEvent_t ev0;
    cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
    cudaEventRecord(ev0, (cudaStream_t)stream);
    for (int i = 0; i < h->stages; ++i) cudaStreamWaitEvent(h->st[i], ev0, 0);
    cudaEventDestroy(ev0);

    const uint64_t nch = (m + h->chunk - 1) / h->chunk;
    uint64_t pend_off[kMaxStages] = {}, pend_cnt[kMaxStages] = {};
    bool pend[kMaxStages] = {};
    int rc = BS_OK;
    for (uint64_t c = 0; c < nch && rc == BS_OK; ++c) {
        const int b = (int)(c % (uint64_t)h->stages);
        const uint64_t off = c * h->chunk;
        const uint64_t cnt = (m - off < h->chunk) ? (m - off) : h->chunk;
        cudaStream_t s = h->st[b];
        if (pend[b]) {   // buffer b is reused: finish its previous chunk first
            cudaEventSynchronize(h->done[b]);
            if (!pin_o) memcpy((char*)host_out + pend_off[b] * ob, h->hout[b], pend_cnt[b] * ob);
            pend[b] = false;
        }
        const void* src = (const char*)host_q + off * kb;
        if (!pin_q) {
            memcpy(h->hq[b], src, cnt * kb);
            src = h->hq[b];
        }
        cudaError_t e = cudaMemcpyAsync(h->dq[b], src, cnt * kb, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) { rc = fail_cuda(e, "bs_lookup_host H2D"); break; }
        rc = dispatch_lookup(ix, h->dq[b], cnt, h->dout[b], s, L);
        if (rc != BS_OK) break;
        void* dst = pin_o ? (void*)((char*)host_out + off * ob) : h->hout[b];
        e = cudaMemcpyAsync(dst, h->dout[b], cnt * ob, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) { rc = fail_cuda(e, "bs_lookup_host D2H"); break; }
        cudaEventRecord(h->done[b], s);
        pend[b] = true;
        pend_off[b] = off;
        pend_cnt[b] = cnt;
    }
    for (int b = 0; b < h->stages; ++b) {
        cudaError_t e = cudaStreamSynchronize(h->st[b]);
        if (e != cudaSuccess && rc == BS_OK) rc = fail_cuda(e, "bs_lookup_host sync");
        if (pend[b] && rc == BS_OK && !pin_o)
            memcpy((char*)host_out + pend_off[b] * ob, h->hout[b], pend_cnt[b] * ob);
    }
    return rc;
}
