// api.cu — the C ABI of libbs.so (include/bs.h): validation, index ownership,
// build orchestration and variant dispatch.  Host code only; the kernels live
// in naive.cu / opt.cu / kary.cu / build.cu.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>

#include "bs.h"
#include "index.h"

namespace bs {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int fail_cuda(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    return fail(e == cudaErrorMemoryAllocation ? BS_ERR_OOM : BS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static bool reserved_zero(const uint32_t* r, int cnt) {
    for (int i = 0; i < cnt; ++i)
        if (r[i]) return false;
    return true;
}

// true if p is device (or managed) memory of `device`: bs_lookup takes GPU-resident
// buffers only ("all data GPU-resident"); a host pointer would fault
// asynchronously inside the kernel.  One driver query per buffer and call
// (a host-side table lookup, well under the launch overhead).
bool device_accessible(const void* p, int device) {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) { cudaGetLastError(); return false; }
    if (pa.type == cudaMemoryTypeManaged) return true;
    return pa.type == cudaMemoryTypeDevice && pa.device == device;
}

// ---- launch planning (params.h plan_grid) ----
namespace {
struct KernelEntry {
    int max_threads = 0;
    int smem_set = -1;        // dynamic shared memory limit set so far
    int carve_set = -1;       // carve-out set so far
    uint32_t occ_threads = 0, occ_smem = 0;
    int occ = -1;             // occupancy of (occ_threads, occ_smem)
};
std::mutex g_plan_mu;
std::unordered_map<uint64_t, std::unordered_map<const void*, KernelEntry>> g_plans;   // device -> kernel
}  // namespace

cudaError_t plan_grid(const void* kern, uint32_t threads, uint32_t smem, Grid grid, uint64_t need, int carveout_pct,
                      uint64_t* blocks, bool* uns) {
    *blocks = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_plan_mu);
    KernelEntry& k = g_plans[(uint64_t)dev][kern];
    if (k.max_threads == 0) {
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, kern);
        if (e != cudaSuccess) return e;
        k.max_threads = fa.maxThreadsPerBlock;
    }
    if ((int)threads > k.max_threads || threads == 0 || threads % 32) { *uns = true; return cudaSuccess; }
    if ((int)smem > k.smem_set) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k.smem_set = (int)smem;
    }
    if (carveout_pct >= 0 && carveout_pct != k.carve_set) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct);
        if (e != cudaSuccess) return e;
        k.carve_set = carveout_pct;
        k.occ = -1;
    }
    uint64_t g = need;
    if (grid.sched_static) {
        int occ = (int)grid.ctas_per_sm;
        if (occ == 0) {
            if (k.occ < 0 || k.occ_threads != threads || k.occ_smem != smem) {
                e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k.occ, kern, (int)threads, smem);
                if (e != cudaSuccess) { k.occ = -1; return e; }
                k.occ_threads = threads;
                k.occ_smem = smem;
            }
            occ = k.occ;
        }
        if (occ < 1) { *uns = true; return cudaSuccess; }
        g = (uint64_t)grid.sm_count * (uint64_t)occ;
    }
    if (g > need) g = need;
    if (g == 0) g = 1;
    if (g > 0x7FFFFFFFull) g = 0x7FFFFFFFull;
    *blocks = g;
    return cudaSuccess;
}


static bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

static uint32_t pow2_at_least(uint32_t x) {
    uint32_t w = 1;
    while (w < x) w <<= 1;
    return w;
}

thread_local const void* t_adopt_keys = nullptr;

static void free_index(Index* ix) {
    if (!ix) return;
    if (ix->d_keys) cudaFree(ix->d_keys);
    if (ix->d_tab) cudaFree(ix->d_tab);
    if (ix->d_sep) cudaFree(ix->d_sep);
    if (ix->d_img) cudaFree(ix->d_img);
    if (ix->d_img64) cudaFree(ix->d_img64);
    if (ix->d_flat) cudaFree(ix->d_flat);
    if (ix->d_flat64) cudaFree(ix->d_flat64);
    if (ix->d_flatimg) cudaFree(ix->d_flatimg);
    if (ix->d_bk) cudaFree(ix->d_bk);
    destroy_host_ctx(ix);
    destroy_dist_state(ix);
    destroy_peer_state(ix);
    delete ix;
}

// Offset-search level structure (DESIGN.md §"Pinned table").
static void compute_levels(Index* ix) {
    const uint64_t n = ix->n;
    ix->s0 = (n >= 2) ? lpow2(n - 1) : 0;
    ix->levels = 0;
    if (n < 2) return;
    uint32_t L = 0;
    for (uint64_t s = ix->s0; s > 0; s >>= 1) ++L;
    ix->levels = L;
    uint64_t acc = 0;
    for (uint32_t d = 0; d < L; ++d) {
        const uint64_t sd = ix->s0 >> d;
        const uint64_t F = (n - 1) / sd;
        ix->valid_all[d] = (F + 1) / 2;      // k < valid_d  <=>  (2k+1) s_d <= n-1
        ix->base_all[d] = acc;
        acc += ix->valid_all[d];
    }
    ix->base_all[L] = acc;                   // == n-1
}

// Choose D / P for a table prefix of at most `entries` entries.
void table_prefix(const Index* ix, uint64_t entries, bool partial, uint32_t* D, uint32_t* P) {
    uint32_t d = 0;
    while (d < ix->levels && ix->base_all[d + 1] <= entries) ++d;
    uint64_t p = 0;
    if (partial && d < ix->levels) {
        p = entries - ix->base_all[d];
        if (p > ix->valid_all[d]) p = ix->valid_all[d];
    }
    *D = d;
    *P = (uint32_t)p;
}

// Device time of each build stage (bs_info.build_stage_us): an event pair
// brackets every group of build kernels, so cudaMalloc and host work between
// them are not counted (Fig. 13).
enum BuildStage { kStSort = 0, kStCheck = 1, kStTable = 2, kStSep = 3, kStImg = 4, kStages = 5 };
struct BuildTimer {
    static constexpr int kMax = 24;
    cudaEvent_t a[kMax] = {}, b[kMax] = {};
    int stage[kMax] = {};
    int used = 0, open = -1;
    cudaStream_t st = nullptr;
    void begin(int s) {
        if (used >= kMax) return;
        if (!a[used]) { cudaEventCreate(&a[used]); cudaEventCreate(&b[used]); }
        stage[used] = s;
        cudaEventRecord(a[used], st);
        open = used;
    }
    void end() {
        if (open < 0) return;
        cudaEventRecord(b[open], st);
        ++used;
        open = -1;
    }
    void collect(float* ms) {   // after a stream sync
        for (int i = 0; i < kStages; ++i) ms[i] = 0;
        for (int i = 0; i < used; ++i) {
            float t = 0;
            if (cudaEventElapsedTime(&t, a[i], b[i]) == cudaSuccess) ms[stage[i]] += t;
        }
        cudaGetLastError();
    }
    ~BuildTimer() {
        for (int i = 0; i < kMax; ++i) {
            if (a[i]) cudaEventDestroy(a[i]);
            if (b[i]) cudaEventDestroy(b[i]);
        }
    }
};

static uint64_t chunks_of(const Index* ix) { return (ix->n + ix->kC - 1) / ix->kC; }

static int build_kary_layout(Index* ix, cudaStream_t st, BuildTimer& bt) {
    const uint64_t n = ix->n;
    const uint32_t K = ix->kK, C = ix->kC, W = ix->kW;
    // bottom-up node counts, then reverse to top-first
    uint64_t counts[kMaxKaryLevels + 2];
    uint32_t L = 0;
    uint64_t c = (n + C - 1) / C;           // leaf chunks
    const uint64_t chunks = c;
    while (c > 1) {
        if (L >= (uint32_t)kMaxKaryLevels) return fail(BS_ERR_INVALID, "K-ary tree deeper than %d levels", kMaxKaryLevels);
        c = (c + K - 1) / K;
        counts[L++] = c;
    }
    ix->kL = L;
    const uint32_t kb = ix->kb;
    const uint64_t align_slots = (W * kb >= 128) ? W : (128 / kb);   // level starts 128-B aligned
    uint64_t slot = 0;
    for (uint32_t l = 0; l < L; ++l) {
        const uint64_t nodes = counts[L - 1 - l];
        ix->k_nodes[l] = nodes;
        ix->k_base[l] = slot;
        slot += nodes * W;
        slot = (slot + align_slots - 1) / align_slots * align_slots;
    }
    for (uint32_t l = 0; l < L; ++l) ix->k_next[l] = (l + 1 < L) ? ix->k_nodes[l + 1] : chunks;
    ix->sep_slots = slot;
    if (chunks > 0xFFFFFFFFull) return fail(BS_ERR_INVALID, "n / leaf_chunk must be < 2^32");
    if (L == 0) return BS_OK;
    const size_t bytes = slot * kb + 16;
    cudaError_t e = cudaMalloc(&ix->d_sep, bytes);
    if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(separators)");
    e = cudaMemsetAsync(ix->d_sep, 0xFF, bytes, st);
    if (e != cudaSuccess) return fail_cuda(e, "memset(separators)");
    bt.begin(kStSep);
    e = build_kary_levels(kb, ix->d_keys, n, K, C, W, L, ix->k_base, ix->k_nodes, ix->d_sep, slot, st);
    bt.end();
    if (e != cudaSuccess) return fail_cuda(e, "build_kary_levels");
    // tiered shared-memory image: the longest level prefix whose planes fit one CTA's shared memory
    {
        // levels whose hi-word plane alone fits one CTA's shared memory (kary_mode 6
        // stages only that plane; modes 2/4 also need the lo plane at word 29056
        // and take a shorter prefix at launch)
        const uint64_t cap_words = ((uint64_t)ix->smem_optin - 1024 - 16) / 4;
        uint32_t words = 0, Li = 0;
        for (uint32_t l = 0; l < L; ++l) {
            const uint64_t w = ((ix->k_nodes[l] * (W + 1) + 3) / 4) * 4;   // 16-B multiple per level
            if (words + w > cap_words) break;
            ix->img_base[l] = words;
            words += (uint32_t)w;
            ++Li;
        }
        ix->img_base[Li] = words;
        ix->img_L = Li;
        if (Li > 0) {
            const uint64_t planes = (kb == 8) ? 2 : 1;
            e = cudaMalloc(&ix->d_img, (uint64_t)words * 4 * planes);
            if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(shared image)");
            uint64_t nodes[kMaxKaryLevels];
            for (uint32_t l = 0; l < Li; ++l) nodes[l] = ix->k_nodes[l];
            bt.begin(kStImg);
            e = build_kary_image(kb, ix->d_sep, W, Li, ix->k_base, nodes, ix->img_base, words, ix->d_img, false, st);
            bt.end();
            if (e != cudaSuccess) return fail_cuda(e, "build_kary_image");
        }
    }
    if (kb == 8) {   // 8-B-slot image (kary_mode 3)
        const uint64_t cap_slots = ((uint64_t)ix->smem_optin - 1024 - 16) / 8;
        uint32_t slots = 0, Li = 0;
        for (uint32_t l = 0; l < L; ++l) {
            const uint64_t w = ((ix->k_nodes[l] * (W + 1) + 1) / 2) * 2;   // 16-B multiple per level
            if (slots + w > cap_slots) break;
            ix->img64_base[l] = slots;
            slots += (uint32_t)w;
            ++Li;
        }
        ix->img64_base[Li] = slots;
        ix->img64_L = Li;
        if (Li > 0) {
            e = cudaMalloc(&ix->d_img64, (uint64_t)slots * 8);
            if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(shared image 64)");
            uint64_t nodes[kMaxKaryLevels];
            for (uint32_t l = 0; l < Li; ++l) nodes[l] = ix->k_nodes[l];
            bt.begin(kStImg);
            e = build_kary_image(kb, ix->d_sep, W, Li, ix->k_base, nodes, ix->img64_base, slots, ix->d_img64, true, st);
            bt.end();
            if (e != cudaSuccess) return fail_cuda(e, "build_kary_image(64)");
        }
    }
    {   // flat pinned table: the deepest level (or the leaf chunks, level L) whose
        // node maxima fit a complete Eytzinger tree of 2^D 4-B words in one CTA's
        // shared memory
        const uint64_t cap_words = ((uint64_t)ix->smem_optin - 1024 - 16) / 4;
        uint32_t lt = 0;
        for (uint32_t l = 0; l <= L; ++l) {
            const uint64_t nl = (l < L) ? ix->k_nodes[l] : chunks_of(ix);
            uint32_t D = 2;   // >= 4 slots: the TMA bulk copy moves multiples of 16 B
            while ((1ull << D) - 1 < nl - 1) ++D;
            if ((1ull << D) <= cap_words) lt = l;
        }
        const uint64_t nl = (lt < L) ? ix->k_nodes[lt] : chunks_of(ix);
        uint32_t D = 2;
        while ((1ull << D) - 1 < nl - 1) ++D;
        uint64_t span = C;                                    // keys under one level-lt node
        for (uint32_t l = lt; l < L; ++l) span *= K;
        ix->flat_level = lt;
        ix->flat_M = nl - 1;
        ix->flat_span = span;
        ix->flat_D = D;
        e = cudaMalloc(&ix->d_flat, 4ull << D);
        if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(flat table)");
        if (kb == 8) {
            e = cudaMalloc(&ix->d_flat64, 8ull << D);
            if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(flat table 64)");
        }
        if (kb == 8) {
            // order-preserving 32-bit image: the array's span in 32 bits (keys < 2^32 exact)
            e = cudaStreamSynchronize(st);   // a_first / a_last are on the host
            if (e != cudaSuccess) return fail_cuda(e, "flat image range");
            const uint64_t span_keys = ix->a_last - ix->a_first;
            uint32_t bl = 0;
            for (uint64_t x = span_keys; x; x >>= 1) ++bl;
            ix->flat_fbase = ix->a_first;
            ix->flat_fshift = bl > 32 ? bl - 32 : 0;
        }
        bt.begin(kStImg);
        e = build_flat_table(kb, ix->d_keys, n, span, ix->flat_M, D, ix->d_flat, ix->d_flat64, ix->flat_fbase,
                             ix->flat_fshift, st);
        bt.end();
        if (e != cudaSuccess) return fail_cuda(e, "build_flat_table");
        // the flat level's node image next to the table (one buffer, one TMA
        // stage): mode 7 then descends one shared level below the table
        ix->flat_img_words = 0;
        if (lt < L && lt < ix->img_L && ix->d_img) {
            const uint64_t wl = ix->img_base[lt + 1] - ix->img_base[lt];   // 4-word multiple
            if ((1ull << D) + wl <= cap_words) {
                e = cudaMalloc(&ix->d_flatimg, ((1ull << D) + wl) * 4);
                if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(flat table + level image)");
                e = cudaMemcpyAsync(ix->d_flatimg, ix->d_flat, 4ull << D, cudaMemcpyDeviceToDevice, st);
                if (e == cudaSuccess) {
                    const uint32_t* hi = (const uint32_t*)ix->d_img + ix->img_base[lt];
                    const uint32_t* lo = kb == 8 ? hi + ix->img_base[ix->img_L] : nullptr;   // lo plane follows hi
                    bt.begin(kStImg);
                    e = build_flat_level_image(hi, lo, wl, ix->flat_fbase, ix->flat_fshift,
                                               (uint32_t*)ix->d_flatimg + (1ull << D), st);
                    bt.end();
                }
                if (e != cudaSuccess) return fail_cuda(e, "flat table + level image");
                ix->flat_img_words = (uint32_t)wl;
            }
        }
    }
    return BS_OK;
}

}  // namespace bs

using namespace bs;

extern "C" {

const char* bs_last_error(void) { return g_err.c_str(); }

uint64_t bs_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* bs_version(void) {
    return "libbs 0.1 (sm_100a; naive / opt / kary; arXiv 2506.01576)";
}

// BS_REORDER_BUCKET structures (part.cu).  Fine: buckets of 2^D units of one
// 32-B leaf (D = 15; BS_BUCKET_D = 14 for A/B runs) while that needs <=
// kBkFineMax buckets (n <= 2^27 u64 / 2^28 u32 keys); above, two-level buckets:
// 2^15 units of 16 leaves of 32 B (16 MB of keys per bucket) with one 32-B node of
// 16-bit leaf-maxima images per unit, up to kBkMaxBuckets (n <= 2^31 u64 / 2^32 u32).
// Tables, per-bucket image parameters, nodes, bucket maxima and their directory
// in one allocation.  Not built (the mode reports UNSUPPORTED) above that.
static int build_bucket_layout(Index* ix, cudaStream_t st, BuildTimer& bt) {
    uint32_t D = 15, G = 1;
    if (const char* v = getenv("BS_BUCKET_D")) D = (uint32_t)atoi(v) == 14 ? 14u : 15u;
    const bool force_two = getenv("BS_BUCKET_TWO") && atoi(getenv("BS_BUCKET_TWO")) != 0;
    uint64_t NB = (1ull << D) * (32u / ix->kb);
    uint64_t B = (ix->n + NB - 1) / NB;
    uint32_t LB = 32;
    if (B > kBkFineMax || force_two) {
        // units of 16 leaves of 32 B with a node of 16-bit images relative to the
        // unit (16-MB buckets): per lookup one node sector and one leaf sector.
        // A/B knob BS_BUCKET_G8=1: units of 8 leaves of 64 B with 32-bit node images
        // (the previous layout: one node sector and two leaf sectors)
        D = 15;
        const bool g8 = getenv("BS_BUCKET_G8") && atoi(getenv("BS_BUCKET_G8")) != 0;
        G = g8 ? 8u : 16u;
        LB = g8 ? 64u : 32u;
        NB = ((uint64_t)G << D) * (LB / ix->kb);
        B = (ix->n + NB - 1) / NB;
    }
    if (B > kBkMaxBuckets) return BS_OK;
    cudaError_t e = cudaStreamSynchronize(st);   // a_first / a_last are on the host
    if (e != cudaSuccess) return fail_cuda(e, "bucket tables: sync");
    auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
    const uint64_t o_tab = 0, o_par = al(4 * (B << D)), o_gn = o_par + al(16 * B);
    const uint64_t gn_bytes = G == 16 ? 2 * (B << D) * G : G > 1 ? 4 * (B << D) * G : 0;
    const uint64_t o_mx = o_gn + al(gn_bytes), o_dir = o_mx + al(4 * B);
    const uint64_t total = o_dir + al(2 * ((1u << 13) + 1));
    e = cudaMalloc(&ix->d_bk, total);
    if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(bucket tables)");
    BucketIndex& bi = ix->bk;
    char* p = (char*)ix->d_bk;
    bi.B = B;
    bi.NB = NB;
    bi.D = D;
    bi.G = G;
    bi.LB = LB;
    bi.gbase = ix->a_first;
    const uint64_t span = ix->a_last - ix->a_first;
    uint32_t bl = 0;
    while (bl < 64 && (span >> bl) != 0) ++bl;
    bi.gsh = bl > 32 ? bl - 32 : 0;
    bt.begin(kStImg);
    e = build_bucket_index(ix->kb, ix->d_keys, ix->n, D, G, LB, NB, B, bi.gbase, bi.gsh, (uint32_t*)(p + o_tab),
                           (uint64_t*)(p + o_par), G > 1 ? (uint32_t*)(p + o_gn) : nullptr, (uint32_t*)(p + o_mx),
                           (uint16_t*)(p + o_dir), st);
    bt.end();
    if (e != cudaSuccess) return fail_cuda(e, "build_bucket_index");
    bi.tab = (const uint32_t*)(p + o_tab);
    bi.par = (const uint64_t*)(p + o_par);
    bi.gnode = G > 1 ? (const uint32_t*)(p + o_gn) : nullptr;
    bi.mx = (const uint32_t*)(p + o_mx);
    bi.dir = (const uint16_t*)(p + o_dir);
    ix->bk_bytes = total;
    return BS_OK;
}

int bs_layout_default(bs_layout* l) {
    if (!l) return fail(BS_ERR_INVALID, "bs_layout_default: NULL");
    memset(l, 0, sizeof *l);
    l->struct_size = sizeof(bs_layout);
    l->key_bytes = 8;
    l->out_bytes = 8;
    l->input_sorted = 1;
    l->variant = BS_VARIANT_KARY;
    l->schedule = BS_SCHED_STATIC;
    l->threads = 0;
    l->nreg = 0;
    l->pin_bytes = 0xFFFFFFFFu;
    l->pin_partial = 1;
    l->reorder = BS_REORDER_NONE;
    l->k = 5;
    l->leaf_chunk = 0;   // auto: resolved by bs_build from the array size
    l->ctas_per_sm = 0;
    l->cache_hints = BS_HINT_AUTO;
    l->kary_mode = BS_KARY_MODE_AUTO;
    return BS_OK;
}

int bs_build(const void* keys, uint64_t n, const bs_layout* layout_in, void** out_idx) {
    if (!out_idx) return fail(BS_ERR_INVALID, "bs_build: out_idx is NULL");
    *out_idx = nullptr;
    bs_layout lay;
    if (layout_in) {
        if (layout_in->struct_size != sizeof(bs_layout))
            return fail(BS_ERR_INVALID, "bs_build: layout.struct_size %u != %zu", layout_in->struct_size, sizeof(bs_layout));
        lay = *layout_in;
    } else {
        bs_layout_default(&lay);
    }
    if (!keys) return fail(BS_ERR_INVALID, "bs_build: keys is NULL");
    if (n == 0) return fail(BS_ERR_INVALID, "bs_build: n == 0 (the offset search needs n >= 1, P:65)");
    if (lay.key_bytes != 4 && lay.key_bytes != 8) return fail(BS_ERR_INVALID, "key_bytes must be 4 or 8");
    if (lay.out_bytes != 4 && lay.out_bytes != 8) return fail(BS_ERR_INVALID, "out_bytes must be 4 or 8");
    if (lay.out_bytes == 4 && n >= (1ull << 31)) return fail(BS_ERR_INVALID, "out_bytes = 4 requires n < 2^31");
    if (lay.variant > BS_VARIANT_KARY) return fail(BS_ERR_INVALID, "unknown variant %u", lay.variant);
    if (lay.schedule > BS_SCHED_STATIC) return fail(BS_ERR_INVALID, "unknown schedule %u", lay.schedule);
    if (lay.reorder > BS_REORDER_BUCKET) return fail(BS_ERR_INVALID, "unknown reorder %u", lay.reorder);
    if (lay.kary_mode > BS_KARY_MODE_AUTO) return fail(BS_ERR_INVALID, "unknown kary_mode %u", lay.kary_mode);
    if (lay.k < 2 || lay.k > 33) return fail(BS_ERR_INVALID, "K must be in [2, 33]");
    if (lay.leaf_chunk != 0 && (!is_pow2(lay.leaf_chunk) || lay.leaf_chunk > 256))
        return fail(BS_ERR_INVALID, "leaf_chunk must be 0 (auto) or a power of two <= 256");
    if (!reserved_zero(lay.reserved, 6)) return fail(BS_ERR_INVALID, "layout.reserved must be zero");
    if (lay.threads > 1024 || lay.threads % 32) return fail(BS_ERR_INVALID, "threads must be a multiple of 32 <= 1024");

    // bs_merge hands over its merged buffer (allocated with the padding below)
    const bool adopt = t_adopt_keys != nullptr && t_adopt_keys == keys && lay.input_sorted;
    t_adopt_keys = nullptr;
    Index* ix = new Index();
    // an adopted buffer (bs_merge / bs_erase) is the index's from here on, so
    // every failure path below frees it through free_index
    if (adopt) ix->d_keys = const_cast<void*>(keys);
    ix->layout = lay;
    ix->n = n;
    ix->kb = lay.key_bytes;
    ix->ob = lay.out_bytes;
    int rc = BS_OK;
    cudaError_t e;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    BuildTimer bt;
    int* d_flag = nullptr;
    const size_t abytes = n * ix->kb;

    e = cudaGetDevice(&ix->device);
    if (e != cudaSuccess) { rc = fail_cuda(e, "cudaGetDevice"); goto done; }
    // the caller's keys may still be in flight on any of its streams (bs_build
    // takes no stream): wait for the device before reading them
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { rc = fail_cuda(e, "bs_build: device synchronisation"); goto done; }
    {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, ix->device); ix->sm_count = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, ix->device); ix->smem_optin = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ix->device); ix->smem_per_sm = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, ix->device); ix->l2_bytes = v;
    }
    ix->hints_requested = ix->layout.cache_hints;
    ix->kary_mode_requested = ix->layout.kary_mode;
    if (ix->layout.kary_mode == BS_KARY_MODE_AUTO) {
        // the pinned Eytzinger table + one shared node level (7) is the fastest
        // thread-per-lookup schedule at every measured size (profiles/r1s3af_*,
        // r1s3ag_*: config 3 +1.8 % sustained over 6, config 2 +22 %)
        ix->layout.kary_mode = 7u;
    }
    if (ix->layout.cache_hints & BS_HINT_AUTO) {
        const uint64_t l2 = ix->l2_bytes ? (uint64_t)ix->l2_bytes : (126ull << 20);
        ix->layout.cache_hints = BS_HINT_STREAM_EVICT_FIRST | BS_HINT_SEP_EVICT_LAST |
                                 ((uint64_t)abytes > 2 * l2 ? BS_HINT_LEAF_EVICT_FIRST : 0u);
    }
    e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e != cudaSuccess) { rc = fail_cuda(e, "cudaStreamCreate"); goto done; }
    bt.st = st;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);

    // ---- the sorted array ----
    // +256 keys of MAX padding: leaf chunks (C <= 256) may be read whole with vector loads
    if (!adopt) {
        e = cudaMalloc(&ix->d_keys, abytes + 256 * ix->kb + 16);
        if (e != cudaSuccess) { rc = fail_cuda(e, "cudaMalloc(keys)"); goto done; }
    }
    e = cudaMemsetAsync((char*)ix->d_keys + abytes, 0xFF, 256 * ix->kb + 16, st);
    if (e != cudaSuccess) { rc = fail_cuda(e, "memset(pad)"); goto done; }
    {
        cudaPointerAttributes pa;
        const bool dev = cudaPointerGetAttributes(&pa, keys) == cudaSuccess &&
                         (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
        cudaGetLastError();
        if (lay.input_sorted) {
            if (!adopt) {
                e = cudaMemcpyAsync(ix->d_keys, keys, abytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
                if (e != cudaSuccess) { rc = fail_cuda(e, "copy keys"); goto done; }
            }
            e = cudaMallocAsync((void**)&d_flag, sizeof(int), st);
            if (e != cudaSuccess) { rc = fail_cuda(e, "cudaMalloc(flag)"); goto done; }
            cudaMemsetAsync(d_flag, 0, sizeof(int), st);
            bt.begin(kStCheck);
            e = build_check_sorted(ix->kb, ix->d_keys, n, d_flag, st);
            bt.end();
            if (e != cudaSuccess) { rc = fail_cuda(e, "check_sorted"); goto done; }
            int flag = 0;
            cudaMemcpyAsync(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st);
            e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) { rc = fail_cuda(e, "check_sorted sync"); goto done; }
            if (flag) { rc = fail(BS_ERR_NOT_SORTED, "bs_build: input_sorted = 1 but keys are not ascending"); goto done; }
        } else {
            void* tmp = nullptr;
            e = cudaMallocAsync(&tmp, abytes, st);
            if (e != cudaSuccess) { rc = fail_cuda(e, "cudaMalloc(sort tmp)"); goto done; }
            e = cudaMemcpyAsync(tmp, keys, abytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
            bt.begin(kStSort);
            if (e == cudaSuccess) e = build_sort_keys(ix->kb, tmp, ix->d_keys, n, st);
            bt.end();
            cudaFreeAsync(tmp, st);
            if (e != cudaSuccess) { rc = fail_cuda(e, "radix sort"); goto done; }
        }
        e = cudaMemcpyAsync(&ix->a_last, (const char*)ix->d_keys + (n - 1) * ix->kb, ix->kb, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) { rc = fail_cuda(e, "read a[n-1]"); goto done; }
        e = cudaMemcpyAsync(&ix->a_first, ix->d_keys, ix->kb, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) { rc = fail_cuda(e, "read a[0]"); goto done; }
    }

    // ---- level-major pinned table (§4.2) ----
    compute_levels(ix);
    {
        uint64_t cap = (uint64_t)ix->smem_optin / ix->kb;
        if (lay.pin_bytes != 0xFFFFFFFFu) cap = lay.pin_bytes / ix->kb;
        uint64_t entries = (n >= 2) ? (n - 1) : 0;
        if (entries > cap) entries = cap;
        ix->tab_entries = entries;
        if (entries) {
            e = cudaMalloc(&ix->d_tab, entries * ix->kb + 16);
            if (e != cudaSuccess) { rc = fail_cuda(e, "cudaMalloc(table)"); goto done; }
            uint32_t bases[kMaxLevels + 1];
            for (uint32_t d = 0; d <= ix->levels; ++d) bases[d] = (uint32_t)(ix->base_all[d] < 0xFFFFFFFFull ? ix->base_all[d] : 0xFFFFFFFFu);
            bt.begin(kStTable);
            e = build_pinned_table(ix->kb, ix->d_keys, n, ix->s0, ix->levels, bases, ix->d_tab, entries, st);
            bt.end();
            if (e != cudaSuccess) { rc = fail_cuda(e, "build_pinned_table"); goto done; }
        }
    }

    // ---- K-ary separator levels (§5) ----
    ix->kK = lay.k;
    ix->leaf_chunk_requested = lay.leaf_chunk;
    if (lay.leaf_chunk == 0) {
        // the smallest leaf of 32 / 64 / 128 bytes whose bottom separator level
        // (one key per leaf) stays within L2/6, else one 128-B line: small
        // arrays read one 32-B sector per lookup, large ones keep the separator
        // levels L2-resident (measured optima at every size: profiles/r1s3x_*)
        const uint64_t l2 = ix->l2_bytes ? (uint64_t)ix->l2_bytes : (126ull << 20);
        uint32_t leaf_bytes = 128;
        for (uint32_t b = 32; b < 128; b <<= 1)
            if ((uint64_t)abytes / b * ix->kb <= l2 / 6) { leaf_bytes = b; break; }
        lay.leaf_chunk = leaf_bytes / ix->kb;
        ix->layout.leaf_chunk = lay.leaf_chunk;
    }
    ix->kC = lay.leaf_chunk;
    ix->kW = pow2_at_least(lay.k - 1 < 2 ? 2 : lay.k - 1);
    if (ix->kW > 32) { rc = fail(BS_ERR_INVALID, "K - 1 must be <= 32"); goto done; }
    if (lay.variant == BS_VARIANT_KARY) {
        rc = build_kary_layout(ix, st, bt);
        if (rc != BS_OK) goto done;
        ix->kary_built = true;
    }

    // ---- per-bucket pinned tables for BS_REORDER_BUCKET (part.cu) ----
    rc = build_bucket_layout(ix, st, bt);
    if (rc != BS_OK) goto done;

    cudaEventRecord(e1, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { rc = fail_cuda(e, "bs_build sync"); goto done; }
    {
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ix->build_ms = ms;
        bt.collect(ix->build_stage_ms);
    }

done:
    if (d_flag) { cudaFreeAsync(d_flag, st); }
    if (st) { cudaStreamSynchronize(st); cudaStreamDestroy(st); }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (rc != BS_OK) { free_index(ix); return rc; }
    *out_idx = ix;
    return BS_OK;
}

void bs_destroy(void* idx) { free_index((Index*)idx); }

int bs_launch_default(const void* idx, bs_launch* l) {
    if (!idx || !l) return fail(BS_ERR_INVALID, "bs_launch_default: NULL");
    const Index* ix = (const Index*)idx;
    memset(l, 0, sizeof *l);
    l->struct_size = sizeof(bs_launch);
    l->variant = ix->layout.variant;
    l->schedule = ix->layout.schedule;
    l->threads = ix->layout.threads;
    l->nreg = ix->layout.nreg;
    l->reorder = ix->layout.reorder;
    l->pin_partial = ix->layout.pin_partial;
    l->ctas_per_sm = ix->layout.ctas_per_sm;
    l->cache_hints = ix->layout.cache_hints;
    l->use_pinned = ix->layout.pin_bytes != 0;
    l->kary_mode = ix->layout.kary_mode;
    return BS_OK;
}

static int lookup_impl(const void* idx, const void* queries, uint64_t m, void* out, void* stream,
                       const bs_launch* launch, void* ws, uint64_t ws_bytes) {
    if (!idx) return fail(BS_ERR_INVALID, "bs_lookup: idx is NULL");
    const Index* ix = (const Index*)idx;
    bs_launch L;
    if (launch) {
        if (launch->struct_size != sizeof(bs_launch)) return fail(BS_ERR_INVALID, "bs_launch.struct_size mismatch");
        L = *launch;
    } else {
        bs_launch_default(idx, &L);
    }
    if (L.kary_mode > 7) return fail(BS_ERR_INVALID, "bs_lookup: unknown kary_mode %u", L.kary_mode);
    if (L.reorder > BS_REORDER_BUCKET) return fail(BS_ERR_INVALID, "bs_lookup: unknown reorder %u", L.reorder);
    if (m == 0) return BS_OK;
    if (!queries || !out) return fail(BS_ERR_INVALID, "bs_lookup: NULL queries/out with m > 0");
    const uintptr_t q0 = (uintptr_t)queries, q1 = q0 + m * ix->kb;
    const uintptr_t o0 = (uintptr_t)out, o1 = o0 + m * ix->ob;
    if (q0 < o1 && o0 < q1) return fail(BS_ERR_INVALID, "bs_lookup: out overlaps queries");
    if (q0 % ix->kb || o0 % ix->ob) return fail(BS_ERR_INVALID, "bs_lookup: misaligned queries/out");
    if (!device_accessible(queries, ix->device) || !device_accessible(out, ix->device))
        return fail(BS_ERR_INVALID, "bs_lookup: queries/out must be device memory of the index's GPU "
                                    "(host buffers: bs_lookup_host)");
    if (L.reorder == BS_REORDER_GLOBAL) {
        uint64_t need = 0;
        if (!part_workspace_bytes(ix->n, m, ix->kb, ix->ob, (uint32_t)ix->sm_count, &need))
            return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_GLOBAL: needs n <= 2^26 keys and m < 2^32");
        if (!ws) return fail(BS_ERR_INVALID, "BS_REORDER_GLOBAL needs a workspace: bs_lookup_ws");
        if (ws_bytes < need)
            return fail(BS_ERR_INVALID, "bs_lookup_ws: workspace of %llu B < %llu B", (unsigned long long)ws_bytes,
                        (unsigned long long)need);
        if (!device_accessible(ws, ix->device)) return fail(BS_ERR_INVALID, "bs_lookup_ws: ws must be device memory");
        bool uns = false;
        cudaError_t e = launch_part_global(ix->kb, ix->ob, ix->d_keys, ix->n, queries, m, out,
                                           (L.cache_hints & BS_HINT_STREAM_EVICT_FIRST) ? 1u : 0u, ws, ws_bytes,
                                           (uint32_t)ix->sm_count, (cudaStream_t)stream, &uns);
        if (uns) return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_GLOBAL: not supported for this index / batch");
        if (e != cudaSuccess) return fail_cuda(e, "global partition launch");
        return BS_OK;
    }
    if (L.reorder == BS_REORDER_BUCKET) {
        uint64_t need = 0;
        if (!ix->bk.mx || !bucket_workspace_bytes(ix->bk.B, m, ix->kb, ix->ob, (uint32_t)ix->sm_count, &need))
            return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_BUCKET: needs n <= %llu keys and m < 2^32",
                        (unsigned long long)bucket_max_keys(ix->kb));
        if (!ws) return fail(BS_ERR_INVALID, "BS_REORDER_BUCKET needs a workspace: bs_lookup_ws");
        if (ws_bytes < need)
            return fail(BS_ERR_INVALID, "bs_lookup_ws: workspace of %llu B < %llu B", (unsigned long long)ws_bytes,
                        (unsigned long long)need);
        if (!device_accessible(ws, ix->device)) return fail(BS_ERR_INVALID, "bs_lookup_ws: ws must be device memory");
        bool uns = false;
        uint32_t chunk = 0;
        if (const char* v = getenv("BS_BUCKET_CHUNK")) chunk = (uint32_t)atoi(v);
        const uint32_t hint = (L.cache_hints & BS_HINT_STREAM_EVICT_FIRST) ? 1u : 0u;
        cudaStream_t s = (cudaStream_t)stream;
        const char* kv = getenv("BS_BUCKET_KARY");
        const bool kary_search = kv && atoi(kv) != 0;
        if (!kary_search) {   // the whole pipeline in part.cu
            cudaError_t e = launch_bucket(ix->kb, ix->ob, ix->bk, ix->d_keys, ix->n, queries, m, out, hint, chunk, ws,
                                          ws_bytes, (uint32_t)ix->sm_count, s, &uns, 0, nullptr);
            if (uns) return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_BUCKET: not supported for this index / batch");
            if (e != cudaSuccess) return fail_cuda(e, "bucket partition launch");
            return BS_OK;
        }
        // A/B (BS_BUCKET_KARY=1): partition, the index's own kernel over the
        // partitioned batch (its array accesses move through one slice at a time),
        // then back to query order
        BucketRun run;
        cudaError_t e = launch_bucket(ix->kb, ix->ob, ix->bk, ix->d_keys, ix->n, queries, m, out, hint, chunk, ws,
                                      ws_bytes, (uint32_t)ix->sm_count, s, &uns, 1, &run);
        if (uns) return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_BUCKET: not supported for this index / batch");
        if (e != cudaSuccess) return fail_cuda(e, "bucket partition launch");
        bs_launch Lk = L;
        Lk.reorder = BS_REORDER_NONE;
        // the partitioned batch reuses each leaf line while its slice is worked
        // on: leaves must not be marked evict_first (the default for arrays > 2 L2)
        Lk.cache_hints &= ~BS_HINT_LEAF_EVICT_FIRST;
        // one persistent launch over the whole partitioned batch.  Measured
        // (config 4, 16-MB buckets): 39 ms for this kernel; a warp-ticket schedule
        // that keeps every warp within one chunk of the batch front cut its DRAM
        // reads from 109 to 17 B / lookup but ran slower (44 ms: on L2-hot slices
        // it is bound by issue and dependent L2 round trips), as did two lookups
        // per thread (64 ms) and one launch per 2^22 queries
        const int rc = dispatch_lookup(ix, run.rq, m, run.rp, s, Lk);
        if (rc != BS_OK) return rc;
        e = launch_bucket(ix->kb, ix->ob, ix->bk, ix->d_keys, ix->n, queries, m, out, hint, chunk, ws, ws_bytes,
                          (uint32_t)ix->sm_count, s, &uns, 2, nullptr);
        if (e != cudaSuccess) return fail_cuda(e, "bucket unpartition launch");
        return BS_OK;
    }
    return dispatch_lookup(ix, queries, m, out, (cudaStream_t)stream, L);
}

int bs_lookup_ex(const void* idx, const void* queries, uint64_t m, void* out, void* stream, const bs_launch* launch) {
    return lookup_impl(idx, queries, m, out, stream, launch, nullptr, 0);
}

int bs_lookup_ws(const void* idx, const void* queries, uint64_t m, void* out, void* stream, const bs_launch* launch,
                 void* ws, uint64_t ws_bytes) {
    return lookup_impl(idx, queries, m, out, stream, launch, ws, ws_bytes);
}

int bs_workspace_bytes(const void* idx, uint64_t m, const bs_launch* launch, uint64_t* bytes) {
    if (!idx || !bytes) return fail(BS_ERR_INVALID, "bs_workspace_bytes: NULL");
    const Index* ix = (const Index*)idx;
    bs_launch L;
    if (launch) {
        if (launch->struct_size != sizeof(bs_launch)) return fail(BS_ERR_INVALID, "bs_launch.struct_size mismatch");
        L = *launch;
    } else {
        bs_launch_default(idx, &L);
    }
    *bytes = 0;
    if (L.reorder == BS_REORDER_BUCKET) {
        if (!ix->bk.mx || !bucket_workspace_bytes(ix->bk.B, m, ix->kb, ix->ob, (uint32_t)ix->sm_count, bytes))
            return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_BUCKET: needs n <= %llu keys and m < 2^32",
                        (unsigned long long)bucket_max_keys(ix->kb));
        return BS_OK;
    }
    if (L.reorder != BS_REORDER_GLOBAL) return BS_OK;
    if (!part_workspace_bytes(ix->n, m, ix->kb, ix->ob, (uint32_t)ix->sm_count, bytes))
        return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_GLOBAL: needs n <= 2^26 keys and m < 2^32");
    return BS_OK;
}

int bs_lookup(const void* idx, const void* queries, uint64_t m, void* out, void* stream) {
    return bs_lookup_ex(idx, queries, m, out, stream, nullptr);
}

int bs_index_info(const void* idx, bs_info* info) {
    if (!idx || !info) return fail(BS_ERR_INVALID, "bs_index_info: NULL");
    const Index* ix = (const Index*)idx;
    memset(info, 0, sizeof *info);
    info->struct_size = sizeof(bs_info);
    info->key_bytes = ix->kb;
    info->out_bytes = ix->ob;
    info->n = ix->n;
    info->array_bytes = ix->n * ix->kb;
    info->pinned_entries = ix->tab_entries;
    uint32_t D = 0, P = 0;
    uint64_t budget = ix->tab_entries;
    table_prefix(ix, budget, ix->layout.pin_partial != 0, &D, &P);
    info->pinned_levels = D;
    info->pinned_partial = P;
    info->search_levels = ix->levels;
    info->kary_levels = ix->kL;
    info->k = ix->kK;
    info->leaf_chunk = ix->kC;
    info->node_slots = ix->kW;
    info->separator_slots = ix->kary_built ? ix->sep_slots : 0;
    info->separator_bytes = info->separator_slots * ix->kb;
    info->kary_smem_levels = ix->kary_built ? kary_smem_levels(ix, nullptr) : 0;
    info->footprint_bytes = info->array_bytes + ix->tab_entries * ix->kb + info->separator_bytes;
    if (ix->d_img) info->footprint_bytes += (uint64_t)ix->img_base[ix->img_L] * 4 * (ix->kb == 8 ? 2 : 1);
    if (ix->d_img64) info->footprint_bytes += (uint64_t)ix->img64_base[ix->img64_L] * 8;
    if (ix->d_flat) info->footprint_bytes += (1ull << ix->flat_D) * (ix->d_flat64 ? 12 : 4);
    if (ix->d_flatimg) info->footprint_bytes += ((1ull << ix->flat_D) + ix->flat_img_words) * 4;
    info->footprint_bytes += ix->bk_bytes;
    info->build_ms = ix->build_ms;
    for (int i = 0; i < 5; ++i) info->build_stage_us[i] = (uint32_t)(ix->build_stage_ms[i] * 1000.0f + 0.5f);
    info->sm_count = ix->sm_count;
    info->smem_per_cta_opt = (uint32_t)ix->last_opt_smem;
    info->smem_per_cta_kary = (uint32_t)ix->last_kary_smem;
    return BS_OK;
}

int bs_export(const void* idx, int what, void* dst, uint64_t cap, uint64_t* written) {
    if (!idx || !dst || !written) return fail(BS_ERR_INVALID, "bs_export: NULL");
    const Index* ix = (const Index*)idx;
    const void* src = nullptr;
    uint64_t bytes = 0;
    switch (what) {
        case BS_EXPORT_SORTED: src = ix->d_keys; bytes = ix->n * ix->kb; break;
        case BS_EXPORT_PINNED: src = ix->d_tab; bytes = ix->tab_entries * ix->kb; break;
        case BS_EXPORT_KARY:
            if (!ix->kary_built) return fail(BS_ERR_UNSUPPORTED, "bs_export: K-ary levels not built");
            src = ix->d_sep; bytes = ix->sep_slots * ix->kb; break;
        default: return fail(BS_ERR_INVALID, "bs_export: unknown structure %d", what);
    }
    if (cap < bytes) return fail(BS_ERR_INVALID, "bs_export: cap %llu < %llu bytes", (unsigned long long)cap, (unsigned long long)bytes);
    *written = 0;
    if (bytes) {
        cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return fail_cuda(e, "bs_export copy");
    }
    *written = bytes;
    return BS_OK;
}

}  // extern "C"
