// index.h — the index object behind the opaque bs_index handle (internal).
#pragma once
#include <cstdint>
#include <atomic>
#include <mutex>

#include <cuda_runtime.h>

#include "bs.h"
#include "common.cuh"
#include "params.h"

namespace bs {

struct HostCtx;    // bs_lookup_host staging (host.cu)
struct DistState;  // multi-GPU exchange state (dist.cu)
struct PeerState;  // fused peer-memory routing state (peer.cu)

// per-call arguments of the g1 kernel's peer prologue / epilogue (params.h)
struct PeerLaunch {
    unsigned long long* cursor;
    const unsigned long long* wait;
    unsigned long long target;
    const uint32_t* tag;
    uint64_t* const* ret;
    unsigned long long* const* sig;
    unsigned* done;
    unsigned* err;
    uint64_t base;
    uint32_t P;
    uint32_t shift;   // tag = (src_rank << shift) | src_idx
};

struct Index {
    bs_layout layout{};
    uint32_t hints_requested = 0;    // layout.cache_hints as given (BS_HINT_AUTO before resolution)
    uint32_t kary_mode_requested = 0;  // layout.kary_mode as given (BS_KARY_MODE_AUTO before resolution)
    uint32_t leaf_chunk_requested = 0; // layout.leaf_chunk as given (0 = auto before resolution)
    int device = 0;
    uint32_t kb = 8, ob = 8;
    uint64_t n = 0;
    void* d_keys = nullptr;          // sorted array, n keys (+16 B slack)
    uint64_t a_last = 0, a_first = 0;  // a[n-1], a[0] (low kb bytes valid)

    // offset-search level structure (all levels) and the level-major table prefix
    uint64_t s0 = 0;
    uint32_t levels = 0;
    uint64_t valid_all[kMaxLevels + 1] = {};
    uint64_t base_all[kMaxLevels + 1] = {};
    void* d_tab = nullptr;
    uint64_t tab_entries = 0;

    // K-ary
    bool kary_built = false;
    void* d_sep = nullptr;
    uint32_t kK = 17, kC = 16, kW = 16, kL = 0;
    uint64_t k_base[kMaxKaryLevels] = {};
    uint64_t k_nodes[kMaxKaryLevels] = {};
    uint64_t k_next[kMaxKaryLevels] = {};
    uint64_t sep_slots = 0;
    // shared-memory image of the top K-ary levels for the tiered schedule:
    // node stride W+1 words (odd: lanes in different nodes reading the same
    // slot fall in different banks); u64 split into a hi-word and a lo-word
    // plane so a probe is one 4-B shared load (the lo word is read only when
    // the hi words tie).  img_base[l] = word offset of level l in a plane.
    void* d_img = nullptr;
    uint32_t img_L = 0;
    uint32_t img_base[kMaxKaryLevels + 1] = {};
    // u64 only: the same image as whole 8-B slots (one plane, node stride W+1
    // slots): one dependent shared load per probe instead of hi then lo
    void* d_img64 = nullptr;
    uint32_t img64_L = 0;
    uint32_t img64_base[kMaxKaryLevels + 1] = {};
    // flat pinned table (kary_mode 7): the maxima of the nodes of K-ary level
    // flat_level except the last node, in Eytzinger order — §4.2's pinned top of a binary
    // search, placed over the K-ary levels.  A binary search over it yields the
    // level-flat_level node directly (~log2 M probes instead of ~1.3x as many
    // node by node).  d_flat: hi words (u64) or keys (u32), staged in shared
    // memory; d_flat64: the exact u64 copy for the tie redo.
    void* d_flat = nullptr;
    void* d_flat64 = nullptr;
    uint64_t flat_M = 0;             // node maxima stored (nodes - 1)
    uint64_t flat_span = 0;          // keys under one flat-level node
    void* d_flatimg = nullptr;       // [flat table (2^flat_D words) | flat level's node image], one stage
    uint32_t flat_img_words = 0;     // words of the level image (0: not built)
    uint32_t flat_level = 0, flat_D = 0;   // Eytzinger slots 1..2^flat_D - 1
    // u64: the flat table and its level image hold F(x) = min((x - flat_fbase) >> flat_fshift,
    // 2^32 - 1) (0 below the base), an order-preserving 32-bit image; flat_fshift makes the
    // array's span fit 32 bits (the hi word when the keys span 2^64; exact when < 2^32)
    uint64_t flat_fbase = 0;
    uint32_t flat_fshift = 32;

    // BS_REORDER_BUCKET: per-bucket pinned tables (part.cu); bk.tab == nullptr: not built
    BucketIndex bk;
    void* d_bk = nullptr;            // one allocation: tab | par | mx | dir
    uint64_t bk_bytes = 0;

    // device
    int sm_count = 148, smem_optin = 232448, smem_per_sm = 233472, l2_bytes = 0;
    double build_ms = 0;
    float build_stage_ms[5] = {};   // sort, sortedness check, pinned table, separators, images + flat table
    // shared memory of the last OPT / K-ary launch (bs_info; atomics: lookups may run concurrently)
    mutable std::atomic<uint64_t> last_opt_smem{0}, last_kary_smem{0};

    // lazily created host-path context
    std::mutex host_mu;
    HostCtx* host = nullptr;

    // multi-GPU
    DistState* dist = nullptr;
    PeerState* peer = nullptr;
};

int fail(int code, const char* fmt, ...);
bool device_accessible(const void* p, int device);
// set by bs_merge right before bs_build(merged, ...): the index adopts that
// device buffer (n keys + 256 keys of padding + 16 B) instead of copying it;
// the index owns it from then on, on success and on failure alike
extern thread_local const void* t_adopt_keys;
int fail_cuda(cudaError_t e, const char* what);
void table_prefix(const Index* ix, uint64_t entries, bool partial, uint32_t* D, uint32_t* P);

// lookup.cu
int dispatch_lookup(const Index* ix, const void* q, uint64_t m, void* out, cudaStream_t s, const bs_launch& L);
int dispatch_kary_peer(const Index* ix, const void* q, uint64_t cap, cudaStream_t s, const bs_launch& L,
                       const PeerLaunch& pl);
uint32_t kary_smem_levels(const Index* ix, uint32_t* bytes_out, uint64_t cap_bytes = 0);
// the layout can run the thread-per-lookup K-ary kernel (kary_mode 6/7), which holds the peer epilogue
bool g1_shape_ok(const Index* ix);

// host.cu / dist.cu
void destroy_host_ctx(Index* ix);
void destroy_dist_state(Index* ix);
void destroy_peer_state(Index* ix);

}  // namespace bs
