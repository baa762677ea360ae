// params.h — kernel parameter blocks and launcher declarations (internal to libbs.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bs {

constexpr int kMaxLevels = 48;      // binary-search levels (n < 2^48)
constexpr int kMaxKaryLevels = 40;  // K-ary internal levels

// Level-major pinned table (DESIGN.md §"Pinned table"; §4.2).
// Level d of the offset search probes positions n-1-(2k+1)*s_d, s_d = s0 >> d,
// s0 = LPOW2(n-1), for k < valid_d; the table stores T[base_d + k] = a[that].
template <class K>
struct OptParams {
    const K* a;           // sorted array (device)
    uint64_t n;
    K a_last;             // a[n-1] (footnote 1: "first entry of the search path")
    uint64_t s0;          // LPOW2(n-1) (first effective step), 0 if n == 1
    uint32_t levels;      // total offset-search levels Dtot = log2(s0)+1 (0 if n == 1)
    const K* tab;         // level-major table (device), 16-B padded
    uint32_t tab_bytes;   // bytes staged into shared memory (0 = no pinning)
    uint32_t D;           // complete levels staged
    uint32_t P;           // entries of level D staged (full-pinning), 0 = steps-pinning
    uint32_t valid[kMaxLevels];
    uint32_t base[kMaxLevels];
    uint64_t evict_step;  // global-phase steps < evict_step use the evict_first hint
    uint64_t l1_step;     // global-phase steps >= l1_step use L1-allocating loads (upper levels that fit L1)
    uint32_t stream_hint; // 1: queries/results with L2 evict_first
    uint32_t leaf_hint;   // 1: deep probes with L2 evict_first
    // block-local reordering (§4.3): bucket = min((q - kmin) >> shift, nbuckets-1)
    K kmin;
    uint32_t shift;
};

template <class KT>
struct KaryParams {
    const KT* a;
    uint64_t n;
    const KT* sep;            // separator levels, top-first, node stride W (device)
    uint32_t L;              // internal levels
    uint32_t K;              // fan-out
    uint32_t C;              // leaf chunk
    uint32_t Ls;             // top levels staged in shared memory
    uint32_t smem_bytes;     // bytes of sep staged (levels 0..Ls-1), 16-B multiple
    uint64_t lvl_base[kMaxKaryLevels];   // element offset of level l (top-first)
    uint32_t nodes_next[kMaxKaryLevels]; // node count of level l+1 (chunks for the last)
    uint32_t stream_hint;
    uint32_t leaf_hint;
    uint32_t sep_hint;       // 1: global separator levels with L2 evict_last
    uint32_t sep_last_end;   // levels >= this get the leaf policy instead (deep levels > L2/2 cumulative)
    // tiered schedule: shared-memory image (Index::d_img), levels 0..Ls-1
    const uint32_t* img;     // hi plane (u64) / the plane (u32), then the lo plane
    uint64_t img_plane_words;// words per plane in global memory
    uint32_t img_base[kMaxKaryLevels];
    uint32_t img_words;      // words of each plane staged (img_base[Ls], 4-word multiple)
    // flat pinned table (kary_mode 7): Eytzinger slots 1..2^flat_D-1 (hi words for u64)
    const uint32_t* flat;    // staged from here (2^flat_D words; slot 0 unused)
    const uint64_t* flat64;  // exact u64 copy (tie redo), u64 keys only
    uint32_t flat_D;
    uint64_t flat_M;         // node maxima in the table (sorted position c < flat_M)
    uint64_t flat_span;      // keys under one node of level Ls: max of node c = a[min((c+1)*span, n) - 1]
    uint32_t flat_img_words; // > 0: the flat level's node image follows the table in smem (mode 7 descends it)
    uint64_t fbase;          // u64 flat image: F(x) = min((x - fbase) >> fshift, 2^32 - 1), 0 below fbase
    uint32_t fshift;
    // fused peer-memory routing (peer.cu, bs_lookup_peer; g1 kernels only).
    // peer_cursor == nullptr: a plain lookup.  Otherwise the kernel first waits
    // until *peer_wait >= peer_wait_target (every rank has routed its queries
    // into this rank's receive window), looks up min(m, *peer_cursor) slots,
    // and stores each result (global rank = peer_base + local lb, miss bit
    // kept) straight into the source rank's return window, slot
    // peer_tag[o] = (src_rank << peer_shift) | src_idx (4 B; peer_shift = 32 -
    // ceil(log2 P), so src_idx < 2^peer_shift).  The last CTA to finish zeroes
    // the cursor and bumps every rank's return counter (*peer_sig[r]).
    unsigned long long* peer_cursor;
    const unsigned long long* peer_wait;
    unsigned long long peer_wait_target;
    const uint32_t* peer_tag;
    uint64_t* const* peer_ret;             // [P] return windows (peer pointers)
    unsigned long long* const* peer_sig;   // [P] return-done counters (peer pointers)
    unsigned int* peer_done;               // local CTA completion counter
    unsigned int* peer_err;                // local error bits (peer_sync.cuh)
    uint64_t peer_base;
    uint32_t peer_P;
    uint32_t peer_shift;
};

// Segment-staged lookup of an ordered batch (seg.cu, BS_REORDER_SORTED)
template <class K>
struct SegParams {
    const K* a;              // sorted array
    uint64_t n;
    const K* q;              // queries (any order; fast when ascending)
    uint64_t m;
    void* out;
    uint32_t ob;
    uint64_t B;              // segments of 2^kSegLog2 keys = ceil(n / S)
    uint32_t stream_hint;    // queries / results with L2 evict_first
};

// ---- launchers (return cudaGetLastError() after the launch) ----
cudaError_t launch_naive(int kb, int ob, const void* a, uint64_t n, const void* q, uint64_t m,
                         void* out, uint32_t threads, cudaStream_t s);


// Grid: sched_static = 0 -> dynamic (one tile / warp-tile set per CTA on the
// hardware scheduler); 1 -> persistent grid of sm_count x ctas_per_sm CTAs
// (ctas_per_sm = 0: as many as are co-resident, from the occupancy API).
struct Grid { uint32_t sched_static, ctas_per_sm, sm_count; };

cudaError_t launch_seg_sorted(int kb, int ob, const void* a, uint64_t n, const void* q, uint64_t m, void* out,
                              uint32_t stream_hint, Grid grid, cudaStream_t s, bool* uns);
// BS_REORDER_GLOBAL (seg.cu): partition -> segment lookups -> unpartition in a caller workspace
bool part_workspace_bytes(uint64_t n, uint64_t m, int kb, int ob, uint32_t sm_count, uint64_t* bytes);
cudaError_t launch_part_global(int kb, int ob, const void* a, uint64_t n, const void* q, uint64_t m, void* out,
                               uint32_t stream_hint, void* ws, uint64_t ws_bytes, uint32_t sm_count, cudaStream_t s,
                               bool* uns);

// BS_REORDER_BUCKET (part.cu): the batch partitioned by key range into buckets whose
// slice of the array stays L2-resident while it is searched.  Each bucket has a
// pinned Eytzinger table of 2^D unit maxima images (built by bs_build, staged by
// TMA).  Fine buckets (n <= 2^27 u64 / 2^28 u32 keys): a unit is one 32-B leaf.
// Two-level buckets (larger n): a unit is 16 leaves of 32 B (16-MB slices), with a
// 32-B global node of the 16 leaf maxima images (16-bit, relative to the unit).
constexpr uint32_t kBkFineMax = 1024;       // most buckets (the partition pass keeps two buckets'
constexpr uint32_t kBkMaxBuckets = 1024;    // state per thread in registers; runs stay long)
constexpr uint32_t kBkChunk = 65536;        // queries per search item (measured at config 3: 8192 3.29 ms,
                                            // 16384 3.08, 32768 2.97, 65536 2.93)
struct BucketIndex {
    uint64_t B = 0;              // buckets
    uint64_t NB = 0;             // keys per bucket (power of two); bucket b = positions [b NB, (b+1) NB)
    uint32_t D = 0;              // table depth: 2^D units per bucket
    uint32_t G = 1;              // leaves per unit: 1 (fine), 16 (two-level; 8 with BS_BUCKET_G8=1)
    uint32_t LB = 32;            // leaf bytes: 32 (64 with BS_BUCKET_G8=1)
    const uint32_t* tab = nullptr;   // [B << D] unit-maxima images, Eytzinger order per bucket
    const uint64_t* par = nullptr;   // [2B] per-bucket image base, shift
    const uint32_t* gnode = nullptr; // two-level: per unit one 32-B node of leaf-maxima images (G = 16:
                                     // 16-bit, relative to the unit; G = 8: 32-bit)
    const uint32_t* mx = nullptr;    // [B] bucket-maxima images under the global image
    const uint16_t* dir = nullptr;   // [2^13 + 1] radix directory over mx
    uint64_t gbase = 0;          // global image: min((x - gbase) >> gsh, 2^32 - 1), 0 below gbase
    uint32_t gsh = 0;
};
struct BucketRun { void* rq = nullptr; void* rp = nullptr; };   // workspace: partitioned queries, their results
cudaError_t build_bucket_index(int kb, const void* a, uint64_t n, uint32_t D, uint32_t G, uint32_t LB, uint64_t NB,
                               uint64_t B, uint64_t gbase, uint32_t gsh, uint32_t* tab, uint64_t* par, uint32_t* gnode,
                               uint32_t* mx, uint16_t* dir, cudaStream_t s);
bool bucket_workspace_bytes(uint64_t B, uint64_t m, int kb, int ob, uint32_t sm_count, uint64_t* bytes);
// largest array a bucket index covers (two-level units of 16 leaves of 32 B)
inline uint64_t bucket_max_keys(uint32_t kb) { return (uint64_t)kBkMaxBuckets * ((8ull << 15) * (64u / kb)); }
// phase 0: the whole pipeline; 1: histogram + partition only (run = the partitioned
// batch, searched by the caller into run->rp: BS_BUCKET_KARY=1 A/B runs); 2: restore
// query order only
// Fused peer return (bs_lookup_peer with layout.reorder = BUCKET, peer.cu): the
// batch is this rank's receive window, its size the received count *m_dev
// (m = min(*m_dev, m)); k_bk_unpart stores the result of window slot s,
// globalised by + base, into ret[tag[s] >> shift][tag[s] & (2^shift - 1)] and
// its last CTA re-arms *cursor and bumps every rank's return counter sig[r].
struct BucketPeer {
    const unsigned long long* m_dev = nullptr;
    uint64_t m_hint = 0;                  // expected batch (sizes the search items)
    const uint32_t* tag = nullptr;
    uint64_t* const* ret = nullptr;       // [P] return windows (device array of peer pointers)
    unsigned long long* const* sig = nullptr;   // [P] return counters
    unsigned long long* cursor = nullptr;
    unsigned* done = nullptr;
    uint64_t base = 0;
    uint32_t P = 1, shift = 32;
};
cudaError_t launch_bucket(int kb, int ob, const BucketIndex& bi, const void* a, uint64_t n, const void* q, uint64_t m,
                          void* out, uint32_t stream_hint, uint32_t chunk, void* ws, uint64_t ws_bytes,
                          uint32_t sm_count, cudaStream_t s, bool* uns, int phase, BucketRun* run,
                          const BucketPeer* peer = nullptr);

// Shared-memory carve-out of a kernel (cudaFuncAttributePreferredSharedMemoryCarveout,
// percent of the SM's 228 KB unified L1/shared array): the smallest that holds the
// resident CTAs' shared memory; the rest stays L1.  Even the K-ary kernels, whose
// global loads do not allocate in L1, need it: L1 also receives the data of every
// load in flight, and a random lookup lives on loads in flight (measured on config
// 3: carve-out 100 % -> 4.99 ms, smallest fitting -> 3.87 ms).
inline int carveout_for(uint32_t smem, uint32_t threads) {
    const uint64_t cap = 228u * 1024u, per = (uint64_t)smem + 1024u;
    uint64_t ctas = 2048u / (threads ? threads : 1u);          // resident CTAs the threads allow
    if (ctas * per > cap) ctas = cap / per;                     // ... and the shared memory
    if (ctas < 1) ctas = 1;
    uint64_t need = ctas * per;
    if (need > cap) need = cap;
    const uint64_t pct = (100u * need + cap - 1) / cap;
    return (int)(pct < 1 ? 1 : pct);
}

// Grid of a lookup launch: `need` blocks of work, or the persistent grid
// (SMs x occupancy) for the static schedule.  The kernel's attributes are queried
// once per (device, kernel); the dynamic-shared-memory limit and the carve-out are
// set only when they change; the occupancy of the last (threads, smem) shape is
// cached.  *uns = true (and no error) if the shape cannot launch.
cudaError_t plan_grid(const void* kern, uint32_t threads, uint32_t smem, Grid grid, uint64_t need, int carveout_pct,
                      uint64_t* blocks, bool* uns);

cudaError_t launch_opt(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                       uint32_t threads, uint32_t nreg, uint32_t reorder, Grid grid,
                       uint32_t smem_bytes, cudaStream_t s, bool* unsupported);
uint32_t opt_smem_extra(int kb, int ob, uint32_t threads, uint32_t nreg, uint32_t reorder);

cudaError_t launch_kary(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                        uint32_t threads, uint32_t W, uint32_t R, Grid grid,
                        uint32_t smem_bytes, cudaStream_t s, bool* unsupported);

// hybrid K-ary: I = waves in flight (divides W), cpl = leaf keys per lane (1, 2, 4)
cudaError_t launch_kary_hybrid(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                               uint32_t threads, uint32_t W, uint32_t I, uint32_t cpl, Grid grid,
                               uint32_t smem_bytes, cudaStream_t s, bool* unsupported);

// tiered K-ary (kary_tiered.cuh): binary search inside shared-memory nodes,
// 16-B vector loads by W*key/16 lanes per lookup below; R = C/W (1, 2, 4),
// I = waves in flight; out word width ob passed at run time
cudaError_t launch_kary_tiered(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                               uint32_t threads, uint32_t W, uint32_t R, uint32_t I, bool pair64, bool pipe,
                               Grid grid, uint32_t smem, cudaStream_t s, bool* unsupported);

// thread-per-lookup K-ary (kary_g1.cuh, kary_mode 6): W*key <= 64 B nodes,
// GL = C*key/32 leaf lanes, IL leaf waves in flight, T lookups per thread in flight
cudaError_t launch_kary_g1(int kb, int ob, const void* params, const void* q, uint64_t m, void* out,
                           uint32_t threads, uint32_t W, uint32_t GL, uint32_t IL, uint32_t T, bool flat,
                           Grid grid, uint32_t smem, cudaStream_t s, bool* unsupported);

// ---- build kernels ----
cudaError_t build_check_sorted(int kb, const void* a, uint64_t n, int* d_flag, cudaStream_t s);
cudaError_t build_pinned_table(int kb, const void* a, uint64_t n, uint64_t s0, uint32_t nlev,
                               const uint32_t* base, void* tab, uint64_t entries, cudaStream_t s);
cudaError_t build_kary_levels(int kb, const void* a, uint64_t n, uint32_t K, uint32_t C, uint32_t W,
                              uint32_t L, const uint64_t* lvl_base, const uint64_t* lvl_nodes,
                              void* sep, uint64_t slots, cudaStream_t s);
cudaError_t build_kary_image(int kb, const void* sep, uint32_t W, uint32_t L, const uint64_t* lvl_base,
                              const uint64_t* lvl_nodes, const uint32_t* img_base, uint64_t plane_words,
                              void* img, bool pair64, cudaStream_t s);
cudaError_t build_flat_table(int kb, const void* a, uint64_t n, uint64_t span, uint64_t M, uint32_t D,
                             void* flat32, void* flat64, uint64_t fbase, uint32_t fshift, cudaStream_t s);
cudaError_t build_flat_level_image(const uint32_t* hi, const uint32_t* lo, uint64_t words, uint64_t fbase,
                                   uint32_t fshift, uint32_t* out, cudaStream_t s);
cudaError_t build_sort_keys(int kb, const void* in, void* out, uint64_t n, cudaStream_t s);

// ---- multi-GPU routing kernels (dist.cu) ----
cudaError_t launch_route(const uint64_t* q, uint64_t m, const uint64_t* shard_max, int P,
                         uint32_t* dest, uint64_t* counts, cudaStream_t s);

}  // namespace bs
