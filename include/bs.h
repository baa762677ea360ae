/*
 * bs.h — C ABI of libbs.so: batched point lookups over a densely packed sorted
 * key array on NVIDIA B200 (sm_100a).  Method: Henneberg & Schuhknecht,
 * "All You Need Is Binary Search! A Practical View on Lightweight Database
 * Indexing on GPUs" (arXiv 2506.01576).  "P:n" below = PAPER.md line n.
 *
 * RESULT CONTRACT (every variant, every knob):
 *   out[i] = lb(q_i)             if a[lb] == q_i           (hit: the rowID)
 *          = lb(q_i) | MISS_BIT  otherwise                 (miss)
 *   lb(q)  = #{ j : a[j] < q }  in [0, n], unsigned compares, a ascending,
 *            duplicates allowed -> first occurrence.
 *   MISS_BIT = 1 << 63 for 8-byte outputs, 1 << 31 for 4-byte outputs.
 *
 * MEMORY: unless stated otherwise pointers are CUDA DEVICE pointers on the
 * current device.  Streams are cudaStream_t passed as void* (NULL = legacy
 * default stream).  No torch / C++ types cross this boundary.
 *
 * ERRORS: every int-returning call returns a bs_status.  Nothing throws or
 * aborts across the ABI.  bs_last_error() returns a thread-local message for
 * the last non-OK status on the calling thread.  Asynchronous device faults
 * of a bs_lookup surface at the caller's next synchronisation (or the next
 * call that synchronises), as with any CUDA launch.
 *
 * THREADING: an index is immutable after bs_build; any number of bs_lookup
 * calls on one index may run concurrently from many host threads / streams.
 * bs_destroy must not race with lookups in flight (caller synchronises).
 */
#ifndef BS_H_
#define BS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BS_OK = 0,
    BS_ERR_INVALID = -1,      /* bad argument (see each call) */
    BS_ERR_UNSUPPORTED = -2,  /* valid but not built into this library / index */
    BS_ERR_OOM = -3,          /* device allocation failed */
    BS_ERR_CUDA = -4,         /* a CUDA runtime call or launch failed */
    BS_ERR_NCCL = -5,         /* an NCCL call failed (multi-GPU entry points) */
    BS_ERR_NOT_SORTED = -6    /* input_sorted = 1 but keys are not ascending */
} bs_status;

typedef enum {
    BS_VARIANT_NAIVE = 0,  /* Listing 1: one thread per lookup, dynamic grid    */
    BS_VARIANT_OPT = 1,    /* §4: scheduling + pinning + reordering ("BS opt")  */
    BS_VARIANT_KARY = 2    /* §5: warp-cooperative K-ary search ("KS")         */
} bs_variant;

typedef enum {
    BS_SCHED_DYNAMIC = 0,  /* hardware block scheduler, one tile per CTA     */
    BS_SCHED_STATIC = 1    /* persistent grid = SMs x ctas_per_sm, strided tiles   */
} bs_schedule;

typedef enum {
    BS_REORDER_NONE = 0,
    BS_REORDER_LOOKUP = 1, /* §4.3 "lookup-reordering": block-local sort, direct stores */
    BS_REORDER_FULL = 2,   /* §4.3 "full-reordering": + inverse permutation before a coalesced
                              store (Listing 2 l.35-39)                                 */
    BS_REORDER_SORTED = 3, /* the batch is ordered (Fig. 1b): segment-staged lookup —
                              per segment of 8192 keys one CTA stages a 32-bit order-preserving
                              image in shared memory and searches its share of the (sorted)
                              batch there.  Any variant's index.  Correct for ANY batch order
                              (queries outside their segment's range take a global
                              bisection); fast only when the batch is ascending.             */
    BS_REORDER_GLOBAL = 4, /* the batch is reordered GLOBALLY (the paper's out-of-place reference
                              point): one partition pass groups the queries by the
                              8192-key segment that holds their answer (records in a caller
                              workspace), the segment-staged lookup runs per segment, one pass
                              restores query order.  Needs bs_lookup_ws; n <= 2^26 keys.     */
    BS_REORDER_BUCKET = 5  /* the batch is partitioned by KEY RANGE (P:131-135's global reorder made
                              coarse) into buckets whose slice of the array stays L2-resident
                              while it is searched: a histogram pass, a partition pass
                              (bucket-major regions, exact offsets), the per-bucket search, one
                              pass restoring query order.  Per bucket bs_build builds a pinned
                              Eytzinger table (§4.2) staged into shared memory by TMA.  Fine
                              buckets (n <= 2^27 u64 / 2^28 u32 keys): the table holds the
                              maxima of 2^15 leaves of 32 B, then one leaf is read (§5).
                              Two-level buckets (larger n, up to 2^31 u64 / 2^32 u32 keys):
                              16 MB of keys; the table holds the maxima of 2^15 units of 8
                              leaves of 64 B, a 32-B node per unit the 8 leaf maxima.  Any
                              variant's index.  Needs bs_lookup_ws.                          */
} bs_reorder;

/* Build-time structure + default launch configuration.
 * Fill with bs_layout_default() and override fields; struct_size guards ABI. */
typedef struct {
    uint32_t struct_size;   /* = sizeof(bs_layout)                                          */
    uint32_t key_bytes;     /* 4 (u32) or 8 (u64); unsigned ordering                 */
    uint32_t out_bytes;     /* 8, or 4 (requires n < 2^31)                                  */
    uint32_t input_sorted;  /* 1: keys already ascending (validated on device);
                               0: the library sorts a copy (unsigned radix sort)            */
    uint32_t variant;       /* bs_variant used by bs_lookup                                 */
    uint32_t schedule;      /* bs_schedule                                                  */
    uint32_t threads;       /* threads per CTA (NBTHREAD); 0 = tuned default         */
    uint32_t nreg;          /* lookups per thread (NREG, Listing 2 l.6) for OPT, interleaved
                               lookup waves per warp for KARY; 0 = tuned default           */
    uint32_t pin_bytes;     /* OPT: shared-memory budget for the pinned top search levels
                               (§4.2); KARY: budget for the top separator levels
                               kept in shared memory (§5.1); 0 = no pinning;
                               0xFFFFFFFF = largest that fits                              */
    uint32_t pin_partial;   /* OPT: 1 = "full-pinning" (partial step M+1), 0 = "steps-pinning" */
    uint32_t reorder;       /* bs_reorder: 1-2 OPT only; 3 (SORTED), 4 (GLOBAL), 5 (BUCKET) any
                               variant                                                      */
    uint32_t k;             /* KARY fan-out K, 2..33 (P:223 A6000 best K = 17)       */
    uint32_t leaf_chunk;    /* KARY leaf chunk C in keys, power of two 1..256; 0 =
                               auto (layout default), resolved by bs_build: the smallest
                               leaf of 32/64/128 B whose bottom separator level fits L2/6,
                               else 128 B (config 3: C = 16; config 2: C = 8)             */
    uint32_t ctas_per_sm;   /* STATIC schedule: resident CTAs per SM; 0 = auto              */
    uint32_t cache_hints;   /* bitmask BS_HINT_*; 0 = plain loads/stores                    */
    uint32_t kary_mode;     /* KARY schedule (same index, same results):
                               0 = warp-cooperative: W lanes per lookup at every level;
                               1 = hybrid: thread per lookup in shared memory (all W slots),
                                   W lanes per lookup in L2/HBM;
                               2 = tiered: thread per lookup with a binary search inside each
                                   shared-memory node, W*key/16 lanes per lookup with 16-B
                                   vector loads in L2/HBM (needs C/W in {1,2,4}, else mode 1);
                               3 = tiered with 8-B shared probes (u64: one slot plane instead
                                   of hi/lo word planes; u32: same as 2);
                               4/5 = 2/3 with a software pipeline across warp-tiles;
                               6 = thread per lookup through the shared AND global separator
                                   levels (node <= 64 B, 256-bit loads), C*key/32 lanes per
                                   lookup for the leaf (needs C*key in 32..256 B, else 2);
                               7 = 6 with the shared levels replaced by a binary search over
                                   a pinned Eytzinger table of one level's node maxima,
                                   then that level's nodes in shared memory when they fit;
                               8 = BS_KARY_MODE_AUTO (layout default), resolved by bs_build
                                   to 7, the fastest at every measured size
                                   (profiles/r1s3af_modes_*, r1s3ag_*)                    */
    uint32_t reserved[6];   /* must be 0                                                    */
} bs_layout;

#define BS_KARY_MODE_AUTO 8u

/* cache_hints bits (B200 L2 eviction-priority hints; not in the paper) */
#define BS_HINT_STREAM_EVICT_FIRST 1u  /* query loads / result stores: L2 evict_first    */
#define BS_HINT_LEAF_EVICT_FIRST 2u    /* deepest probes / K-ary leaves: L2 evict_first  */
#define BS_HINT_SEP_EVICT_LAST 4u      /* K-ary separator levels in global memory: L2 evict_last */
/* Resolved by bs_build (the layout default): STREAM | SEP, plus LEAF when the
 * sorted array exceeds twice the L2 — evict_first on leaves pays only when
 * they cannot stay resident (measured: profiles/r1s3f_hints_*.jsonl). */
#define BS_HINT_AUTO 0x100u

/* Per-call launch override (bs_lookup_ex).  Only launch knobs; the structure
 * built by bs_build (pinned table size, K, C) is fixed.  Field meaning as in
 * bs_layout; 0 in threads/nreg/ctas_per_sm means "index default".           */
typedef struct {
    uint32_t struct_size;   /* = sizeof(bs_launch) */
    uint32_t variant;
    uint32_t schedule;
    uint32_t threads;
    uint32_t nreg;
    uint32_t reorder;
    uint32_t pin_partial;
    uint32_t ctas_per_sm;
    uint32_t cache_hints;
    uint32_t use_pinned;    /* 1: use the pinned table / shared separator levels (if built) */
    uint32_t kary_mode;     /* as bs_layout.kary_mode                                        */
    uint32_t reserved[5];
} bs_launch;

typedef struct {
    uint32_t struct_size;        /* = sizeof(bs_info) */
    uint32_t key_bytes, out_bytes;
    uint64_t n;
    uint64_t footprint_bytes;    /* all device memory owned by the index (Fig. 12) */
    uint64_t array_bytes;        /* n * key_bytes                                         */
    uint64_t pinned_entries;     /* level-major pinned table entries (OPT)                */
    uint32_t pinned_levels;      /* M: complete levels pinned (§4.2)                      */
    uint32_t pinned_partial;     /* entries of level M kept (full-pinning)         */
    uint32_t search_levels;      /* total binary-search steps = floor(log2(n-1)) + 1      */
    uint32_t kary_levels;        /* internal K-ary levels                                 */
    uint32_t k, leaf_chunk, node_slots;
    uint32_t kary_smem_levels;   /* top K-ary levels staged in shared memory              */
    uint64_t separator_slots;    /* K-ary slots incl. padding (node_slots per node)       */
    uint64_t separator_bytes;
    double build_ms;             /* device time from bs_build's first to last stream op (incl. gaps) */
    uint32_t sm_count;
    uint32_t smem_per_cta_opt;   /* dynamic shared memory of the OPT kernel (bytes)       */
    uint32_t smem_per_cta_kary;
    uint32_t build_stage_us[5];  /* device time of each build stage in microseconds, allocation
                                    excluded (Fig. 13): [0] radix sort of unsorted
                                    input, [1] sortedness check of sorted input, [2] pinned table,
                                    [3] K-ary separators, [4] shared-memory images + flat table */
} bs_info;

/* Debug exports (layout-fidelity tests) for bs_export(). */
#define BS_EXPORT_SORTED 0   /* the sorted key array (n keys)                          */
#define BS_EXPORT_PINNED 1   /* the level-major pinned table (pinned_entries keys)     */
#define BS_EXPORT_KARY 2     /* K-ary separator slots, levels top-first (separator_slots) */

/* Fills *l with defaults for u64 keys/outputs: K-ary, K = 5 (the paper's
 * A6000 optimum was K = 17), leaf chunk, schedule and
 * L2 hints left to bs_build (leaf_chunk = 0, kary_mode = BS_KARY_MODE_AUTO,
 * cache_hints = BS_HINT_AUTO: at 2^26 u64 keys they resolve to C = 16, the
 * thread-per-lookup kary_mode 7 and stream + separator hints), largest pin
 * budget, static schedule.  BS_ERR_INVALID if l is NULL. */
int bs_layout_default(bs_layout* l);

/* Fills *l with the per-call defaults stored in idx. */
int bs_launch_default(const void* idx, bs_launch* l);

/*
 * Builds an immutable index over n keys ("sorted input array of size n",
 * P:119 pinned entries, P:213 K-ary separators, built bottom-up).
 *   keys     device OR host pointer to n keys of layout->key_bytes each; the
 *            library copies (and if input_sorted = 0 sorts) them into
 *            library-owned device memory; the caller's buffer is untouched.
 *   n        >= 1 (P:65 needs n-1 >= 0); out_bytes = 4 requires n < 2^31.
 *   layout   see bs_layout; NULL = bs_layout_default().
 *   out_idx  receives the index; NULL on error.
 * Synchronous: waits for all prior work on the device (the keys may have been
 * produced on any stream), returns when the index is ready.  Always builds the pinned
 * table for OPT and the separator levels for KARY; the NAIVE variant needs
 * neither.  Errors: BS_ERR_INVALID (NULL pointers, n == 0, bad widths, K not
 * in [2,33], C not a power of two in [1,256], nonzero reserved fields),
 * BS_ERR_NOT_SORTED, BS_ERR_OOM, BS_ERR_CUDA.
 */
int bs_build(const void* keys, uint64_t n, const bs_layout* layout, void** out_idx);

/*
 * Looks up m queries ("probes ... keys"; §4.4 Listing 2).
 *   idx      from bs_build.
 *   queries  device pointer, m keys of key_bytes (any alignment of the element
 *            type).
 *   m        0 is allowed (no launch, BS_OK).
 *   out      device pointer, m words of out_bytes; must not overlap queries.
 *   stream   cudaStream_t (void*); the call is stream-ordered and
 *            asynchronous: no allocation, no host synchronisation.
 * Errors: BS_ERR_INVALID (NULL idx / pointers with m > 0, overlap, misaligned,
 * or queries / out not device memory of the index's GPU — checked with
 * cudaPointerGetAttributes; host buffers go through bs_lookup_host),
 * BS_ERR_CUDA (launch failure).
 * Kernel attributes, the dynamic shared memory limit, the shared-memory
 * carve-out (all of the unified L1 for the K-ary kernels, whose pinned levels
 * live there) and the occupancy are set / queried once per kernel
 * and shape, not per call.
 */
int bs_lookup(const void* idx, const void* queries, uint64_t m, void* out, void* stream);

/* bs_lookup with per-call launch knobs (variant, schedule, threads, nreg,
 * reorder, pinning use).  BS_ERR_UNSUPPORTED if the requested variant's
 * structure was not built or the knob combination is not compiled in. */
int bs_lookup_ex(const void* idx, const void* queries, uint64_t m, void* out, void* stream,
                 const bs_launch* launch);

/*
 * End-to-end lookup from HOST memory: copies queries host->device, runs the
 * index's default lookup, copies results device->host, in pipelined chunks
 * on internal streams (copy of chunk i+1 overlaps lookup of chunk i and the
 * copy-back of chunk i-1).
 *   host_queries / host_out  host pointers (pinned memory gives full PCIe
 *            bandwidth; pageable memory is staged through internal pinned
 *            buffers).
 *   stream   the call is ordered after prior work on `stream` and returns
 *            when host_out is complete (synchronous).
 * Allocates its staging buffers on first use per index (then reuses them;
 * serialised by an internal mutex).  Errors as bs_lookup, plus BS_ERR_OOM.
 */
int bs_lookup_host(const void* idx, const void* host_queries, uint64_t m, void* host_out,
                   void* stream);

/*
 * Workspace-taking lookup (the BS_REORDER_GLOBAL and BS_REORDER_BUCKET modes,
 * which partition the batch out of place).
 *   bs_workspace_bytes: *bytes = device bytes a bs_lookup_ws call with this
 *     launch (NULL = index defaults) needs for m queries (0 if the mode needs
 *     none; BUCKET: m * (key + out + 4) bytes plus per-CTA / per-tile tables).
 *     BS_ERR_UNSUPPORTED if the mode cannot run on this index (GLOBAL:
 *     n > 2^26 keys; BUCKET: more than 1024 buckets; either: m >= 2^32).
 *   bs_lookup_ws: bs_lookup_ex plus a caller-owned device workspace `ws` of
 *     ws_bytes (no allocation inside; the workspace must not be shared by calls
 *     in flight on other streams).  BS_ERR_INVALID if ws is NULL / too small for
 *     a mode that needs one.  Other modes ignore ws.  Same result contract.
 * bs_lookup / bs_lookup_ex with reorder = BS_REORDER_GLOBAL or BUCKET return
 * BS_ERR_INVALID (no workspace).
 */
int bs_workspace_bytes(const void* idx, uint64_t m, const bs_launch* launch, uint64_t* bytes);
int bs_lookup_ws(const void* idx, const void* queries, uint64_t m, void* out, void* stream, const bs_launch* launch,
                 void* ws, uint64_t ws_bytes);

/* Frees everything the index owns.  NULL-safe.  No lookups may be in flight. */
void bs_destroy(void* idx);

/* Thread-local message for the last non-OK status ("" if none). */
const char* bs_last_error(void);

/* Sizes and structure of an index (Fig. 12 footprint, Fig. 13 build time). */
int bs_index_info(const void* idx, bs_info* info);

/* Copies one internal structure (BS_EXPORT_*) to HOST memory dst of `cap`
 * bytes; *written = bytes copied.  Synchronous.  Test/debug use only.
 * BS_ERR_INVALID if cap is too small, BS_ERR_UNSUPPORTED if not built. */
int bs_export(const void* idx, int what, void* dst, uint64_t cap, uint64_t* written);

/* Batch insert (the paper's outlook, gives no method):
 * builds a NEW index, same layout, over the multiset union of idx's keys and
 * delta_keys (m device keys of idx's key width; delta_sorted = 1 if already
 * ascending, else the library radix-sorts a copy).  The old array and the
 * sorted delta are merged on the device (merge path), then the auxiliary
 * levels are rebuilt.  idx is untouched (destroy it when no lookup on it is in
 * flight); results on *out_idx follow the result contract over the merged
 * array.  Synchronous.  m = 0 clones idx.  Errors: BS_ERR_INVALID,
 * BS_ERR_UNSUPPORTED (multi-GPU index), BS_ERR_NOT_SORTED (delta_sorted = 1
 * but not ascending), BS_ERR_CUDA / BS_ERR_OOM. */
int bs_merge(const void* idx, const void* delta_keys, uint64_t m, int delta_sorted, void** out_idx);

/* Batch delete (same outlook): builds a NEW index, same layout, over
 * idx's keys minus every key equal to one of the m device keys del_keys
 * (set difference: all occurrences of a deleted value go; values not present
 * are ignored; del_sorted = 1 if ascending, else the library sorts a copy).
 * idx is untouched.  Synchronous.  m = 0 clones idx.  Errors: BS_ERR_INVALID
 * (NULL, or every key erased: an index needs n >= 1), BS_ERR_UNSUPPORTED
 * (multi-GPU index), BS_ERR_CUDA / BS_ERR_OOM. */
int bs_erase(const void* idx, const void* del_keys, uint64_t m, int del_sorted, void** out_idx);

/* Library version / build string (arch, commit-independent). */
const char* bs_version(void);

/* Number of kernels this library has launched on its lookup paths (bs_lookup*,
 * bs_lookup_host, bs_lookup_dist, bs_lookup_peer; not bs_build) since it was
 * loaded, all threads and devices.  Read it before and after a region to count
 * the region's launches (bench.py's gpu_launches). */
uint64_t bs_launch_count(void);

/* ------------------------------------------------------------------------
 * Multi-GPU (one process per GPU; BASELINE.json configs 4-5, not in the
 * paper).  REPLICATED: every rank builds the full index; queries are sharded
 * by the caller; no collective on the lookup path.  PARTITIONED: rank r holds
 * the contiguous rank range [base_r, base_r + n_r) of the global sorted
 * array; bs_lookup_dist routes each query to the first shard whose maximum
 * is >= q (else the last shard), looks it up there and returns the GLOBAL
 * result (base + local lb, miss bit kept), in the caller's query order.
 * ---------------------------------------------------------------------- */

#define BS_DIST_REPLICATED 0
#define BS_DIST_PARTITIONED 1

/* Size of the NCCL unique id blob (bytes). */
#define BS_DIST_UID_BYTES 128

/* Rank 0 fills uid (BS_DIST_UID_BYTES host bytes); the caller broadcasts it
 * (e.g. over torch.distributed's store) before every rank calls bs_dist_init. */
int bs_dist_get_uid(void* uid);

/* Creates the NCCL communicator for (rank, world) on the current device.
 * Collective across ranks.  out_comm receives an opaque handle. */
int bs_dist_init(const void* uid, int rank, int world, void** out_comm);

/*
 * Collective: builds this rank's index over its local, ascending keys
 * (device pointer, n_local >= 1) and exchanges shard metadata (maxima and
 * sizes) with ncclAllGather.  mode = BS_DIST_REPLICATED or
 * BS_DIST_PARTITIONED.  max_m_local bounds m_local of later lookups (sizes
 * the exchange buffers, allocated here).  Shards must be globally ordered by
 * rank (max of rank r <= min of rank r+1) in PARTITIONED mode, checked.
 */
int bs_build_dist(void* comm, const void* local_keys, uint64_t n_local, int mode,
                  const bs_layout* layout, uint64_t max_m_local, void** out_idx);

/*
 * Collective in PARTITIONED mode (every rank must call, m_local may be 0):
 * route (k_route) -> count exchange -> query all-to-all (grouped
 * ncclSend/ncclRecv) -> local lookup -> result all-to-all -> unroute.
 * REPLICATED mode: a plain local bs_lookup, no communication.
 * out_local receives global results (out_bytes must be 8 in PARTITIONED).
 */
int bs_lookup_dist(const void* idx, const void* local_queries, uint64_t m_local, void* out_local,
                   void* stream);

/* Destroys the communicator (after all dist indexes using it). NULL-safe. */
void bs_dist_destroy(void* comm);

/* ------------------------------------------------------------------------
 * Fused peer-memory routing (PARTITIONED mode without NCCL; SURVEY §8f f1,
 * BASELINE.json config 5; not in the paper).  Same result contract as
 * bs_lookup_dist in PARTITIONED mode: out_local[i] = base_s + lb_s(q_i)
 * (| bit 63 on a miss), s = first shard whose maximum is >= q_i (else the
 * last).  The exchange runs inside the kernels over CUDA-IPC-mapped peer
 * memory (NVLink / NVSwitch P2P): the route kernel stores each query into
 * its owner's receive window, the K-ary lookup kernel (kary_mode 6/7) stores
 * each result into its source rank's return window, and monotonic device
 * counters replace the host sync and the NCCL all-to-alls.
 *
 * Setup, per rank (one process per GPU; also valid for several processes
 * sharing one GPU, which is how it is tested on a 1-GPU box):
 *   bs_build_peer -> bs_peer_export -> (caller all-gathers the blobs, e.g.
 *   torch.distributed.all_gather_object) -> bs_peer_connect.
 * ---------------------------------------------------------------------- */

/* Bytes of one rank's connection blob (host memory). */
#define BS_PEER_BLOB_BYTES 256

/* Builds this rank's index over its local ascending keys (device pointer,
 * n_local >= 1; layout must give variant KARY and out_bytes 8; layout.reorder
 * = BS_REORDER_BUCKET makes the owner look its receive window up with the
 * key-range partition pipeline, whose unpartition stores the results into
 * the sources' return windows — workspace for recv_capacity queries is
 * allocated here, n_local must fit a bucket index and recv_capacity < 2^32;
 * any other reorder runs the K-ary kernel's peer epilogue) and allocates
 * its IPC-exportable window: receive slots (recv_capacity keys + 4-B return
 * tags, (src_rank << (32 - ceil(log2 world))) | src_idx; recv_capacity 0 =
 * world * max_m_local, which can never overflow) and a return window of
 * max_m_local results.  max_m_local bounds m_local of later lookups and must
 * be < 2^32 and <= 2^(32 - ceil(log2 world)) (2^29 at world 8).
 * Not collective.  Errors: BS_ERR_INVALID (bad rank/world/sizes/layout),
 * BS_ERR_UNSUPPORTED (variant is not KARY), BS_ERR_OOM, plus bs_build's. */
int bs_build_peer(const void* local_keys, uint64_t n_local, const bs_layout* layout, int rank, int world,
                  uint64_t max_m_local, uint64_t recv_capacity, void** out_idx);

/* Writes this rank's connection blob (BS_PEER_BLOB_BYTES host bytes: the
 * window's cudaIpcMemHandle_t, shard size and min/max key). */
int bs_peer_export(const void* idx, void* blob);

/* blobs = world consecutive blobs in rank order (host memory).  Checks that
 * the shards are globally ordered (BS_ERR_NOT_SORTED otherwise), derives each
 * shard's global base rank, maps every peer's window (cudaIpcOpenMemHandle,
 * lazy peer access).  Once per index; not collective, but every rank must
 * connect before any rank calls bs_lookup_peer. */
int bs_peer_connect(void* idx, const void* blobs);

/* Collective (every rank calls it, in the same order, m_local may be 0):
 * route -> lookup -> return, three kernels on `stream`, stream-ordered and
 * asynchronous, no host sync, no allocation.  local_queries: m_local keys;
 * out_local: m_local u64 global results (device pointers, must not overlap
 * the index's windows), or NULL to leave the results in the return window
 * (bs_peer_results; saves one copy, valid until the next call).  A peer that never joins makes the waits time out
 * (after BS_PEER_WAIT_MS from the environment at build time, default 20000;
 * error bit 2 in bs_peer_status, results undefined) instead of hanging the
 * GPU.  Not thread-safe per index. */
int bs_lookup_peer(const void* idx, const void* local_queries, uint64_t m_local, void* out_local, void* stream);

/* *results = device pointer of this rank's return window: after a
 * bs_lookup_peer with out_local == NULL, results[i] is query i's global
 * result once the call's stream work has completed. */
int bs_peer_results(const void* idx, const void** results);

/* Synchronous diagnostic: *err_bits = OR of 1 (a receive window overflowed:
 * recv_capacity too small, queries dropped) and 2 (a wait timed out) since
 * build; *calls (may be NULL) = bs_lookup_peer calls issued. */
int bs_peer_status(const void* idx, uint32_t* err_bits, uint64_t* calls);

#ifdef __cplusplus
}
#endif

#endif /* BS_H_ */
