// lookup.cu — per-call variant dispatch: builds the kernel parameter blocks
// from the index and the launch knobs, sizes shared memory, launches.
#include <cstdlib>
#include <cstring>

#include "index.h"

namespace bs {

static uint32_t round16(uint64_t b) { return (uint32_t)((b + 15) & ~15ull); }

static uint32_t bitlen(uint64_t x) {
    uint32_t b = 0;
    while (x) { ++b; x >>= 1; }
    return b;
}

// shared memory one CTA may use when `c` CTAs share an SM (1 KB per CTA is
// reserved by the system on sm_100)
static uint64_t smem_cap(const Index* ix, uint32_t c) {
    if (c == 0) c = 1;
    uint64_t per = (uint64_t)ix->smem_per_sm / c;
    per = per > 1024 ? per - 1024 : 0;
    if (per > (uint64_t)ix->smem_optin) per = ix->smem_optin;
    return per & ~15ull;
}

uint32_t kary_smem_levels(const Index* ix, uint32_t* bytes_out, uint64_t cap_bytes) {
    if (cap_bytes == 0) cap_bytes = smem_cap(ix, 1) - 16;
    if (ix->layout.pin_bytes != 0xFFFFFFFFu && ix->layout.pin_bytes < cap_bytes) cap_bytes = ix->layout.pin_bytes;
    uint32_t Ls = 0;
    while (Ls < ix->kL) {
        const uint64_t end = (Ls + 1 < ix->kL) ? ix->k_base[Ls + 1] : ix->sep_slots;
        if (end * ix->kb > cap_bytes) break;
        ++Ls;
    }
    if (bytes_out) *bytes_out = Ls ? round16((Ls < ix->kL ? ix->k_base[Ls] : ix->sep_slots) * ix->kb) : 0;
    return Ls;
}

template <class K>
static int run_opt(const Index* ix, const void* q, uint64_t m, void* out, cudaStream_t s, const bs_launch& L) {
    OptParams<K> p;
    memset(&p, 0, sizeof p);
    p.a = (const K*)ix->d_keys;
    p.n = ix->n;
    p.a_last = (K)ix->a_last;
    p.s0 = ix->s0;
    p.levels = ix->levels;
    p.tab = (const K*)ix->d_tab;
    const uint32_t threads = L.threads ? L.threads : 256;
    const uint32_t nreg = L.nreg ? L.nreg : 8;
    if (threads % 32 || threads > 1024) return fail(BS_ERR_INVALID, "threads must be a multiple of 32 <= 1024");
    const uint32_t extra = opt_smem_extra(ix->kb, ix->ob, threads, nreg, L.reorder);
    const uint32_t cps = L.schedule == BS_SCHED_STATIC ? L.ctas_per_sm : 0;
    const uint64_t cap = smem_cap(ix, cps ? cps : 1);
    if (extra > cap) return fail(BS_ERR_UNSUPPORTED, "OPT: tile of %u x %u does not fit shared memory", threads, nreg);
    uint64_t entries = 0;
    if (L.use_pinned && ix->d_tab) {
        uint64_t budget = cap - extra;
        if (ix->layout.pin_bytes != 0xFFFFFFFFu && ix->layout.pin_bytes < budget) budget = ix->layout.pin_bytes;
        entries = budget / ix->kb;
        if (entries > ix->tab_entries) entries = ix->tab_entries;
    }
    uint32_t D = 0, P = 0;
    table_prefix(ix, entries, L.pin_partial != 0, &D, &P);
    if (D >= (uint32_t)kMaxLevels) D = kMaxLevels - 1;
    p.D = D;
    p.P = P;
    for (uint32_t d = 0; d <= D && d < (uint32_t)kMaxLevels; ++d) {
        p.valid[d] = (uint32_t)ix->valid_all[d];
        p.base[d] = (uint32_t)ix->base_all[d];
    }
    const uint64_t used = ix->base_all[D] + P;
    p.tab_bytes = used ? round16(used * ix->kb) : 0;
    // global-phase steps whose levels cannot stay in (half of) L2 get evict_first
    const uint64_t l2 = ix->l2_bytes ? (uint64_t)ix->l2_bytes : (126ull << 20);
    uint64_t es = 1;
    while (es < (32ull * ix->n) / (l2 / 2)) es <<= 1;
    p.evict_step = es;
    // L1-allocating loads for the first global levels whose probe lines fit
    // ~96 KB of L1 (2^d positions per level, one 128-B line each at most)
    {
        const uint64_t lines_total = (ix->n * ix->kb + 127) / 128;
        uint64_t cum = 0, l1s = ~0ull;
        const uint32_t d0 = P ? D + 1 : D;   // first level of the global phase
        for (uint32_t d = d0; d < ix->levels; ++d) {
            const uint64_t lines = d < 63 ? ((1ull << d) < lines_total ? (1ull << d) : lines_total) : lines_total;
            if (cum + lines > 768) break;
            cum += lines;
            l1s = ix->s0 >> d;
        }
        p.l1_step = l1s;
    }
    p.stream_hint = (L.cache_hints & BS_HINT_STREAM_EVICT_FIRST) ? 1 : 0;
    p.leaf_hint = (L.cache_hints & BS_HINT_LEAF_EVICT_FIRST) ? 1 : 0;
    p.kmin = (K)ix->a_first;
    const uint64_t range = (uint64_t)((K)ix->a_last - (K)ix->a_first);
    const uint32_t tb = bitlen(threads * nreg) - 1;
    const uint32_t rb = bitlen(range);
    p.shift = rb > tb ? rb - tb : 0;
    const uint32_t smem = p.tab_bytes + extra;
    ix->last_opt_smem = smem;
    bool uns = false;
    Grid g{L.schedule == BS_SCHED_STATIC ? 1u : 0u, L.ctas_per_sm, (uint32_t)ix->sm_count};
    cudaError_t e = launch_opt(ix->kb, ix->ob, &p, q, m, out, threads, nreg, L.reorder, g, smem, s, &uns);
    if (uns) return fail(BS_ERR_UNSUPPORTED, "OPT: threads=%u nreg=%u reorder=%u not supported", threads, nreg, L.reorder);
    if (e != cudaSuccess) return fail_cuda(e, "OPT launch");
    return BS_OK;
}

template <class K>
static int run_kary(const Index* ix, const void* q, uint64_t m, void* out, cudaStream_t s, const bs_launch& L,
                    const PeerLaunch* pl = nullptr) {
    if (!ix->kary_built) return fail(BS_ERR_UNSUPPORTED, "KARY: index built without K-ary levels (layout.variant != KARY)");
    KaryParams<K> p;
    memset(&p, 0, sizeof p);
    p.a = (const K*)ix->d_keys;
    p.n = ix->n;
    p.sep = (const K*)ix->d_sep;
    p.L = ix->kL;
    p.K = ix->kK;
    p.C = ix->kC;
    for (uint32_t l = 0; l < ix->kL; ++l) {
        p.lvl_base[l] = ix->k_base[l];
        p.nodes_next[l] = (uint32_t)ix->k_next[l];
    }
    const uint32_t W = ix->kW, C = ix->kC;
    const uint32_t GL = C * ix->kb / 32;
    const bool g1 = (L.kary_mode == 6 || L.kary_mode == 7) && W * ix->kb <= 64 && W * ix->kb >= 8 && C * ix->kb >= 32 &&
                    C * ix->kb <= 256;
    if (pl && !g1)
        return fail(BS_ERR_UNSUPPORTED, "bs_lookup_peer: needs the thread-per-lookup K-ary kernel (kary_mode 6/7, "
                                        "W*key <= 64 B, C*key in 32..256 B)");
    if (pl) {
        p.peer_cursor = pl->cursor;
        p.peer_wait = pl->wait;
        p.peer_wait_target = pl->target;
        p.peer_tag = pl->tag;
        p.peer_ret = pl->ret;
        p.peer_sig = pl->sig;
        p.peer_done = pl->done;
        p.peer_err = pl->err;
        p.peer_base = pl->base;
        p.peer_P = pl->P;
        p.peer_shift = pl->shift;
    }
    const bool tiered = !g1 && L.kary_mode >= 2 && C >= W && (C / W == 1 || C / W == 2 || C / W == 4);
    const bool pair64 = (L.kary_mode == 3 || L.kary_mode == 5) && ix->kb == 8;
    const bool pipe = L.kary_mode >= 4;   // 4/5: experimental software-pipelined 2/3
    const uint32_t threads = L.threads ? L.threads : ((tiered || g1) ? 1024 : 512);
    const uint32_t R = L.nreg ? L.nreg : 2;
    const bool stat = L.schedule == BS_SCHED_STATIC;
    uint32_t Ls = 0, sbytes = 0;
    if (stat && L.use_pinned) {
        const uint64_t cap = smem_cap(ix, L.ctas_per_sm ? L.ctas_per_sm : 1) - 16;
        Ls = kary_smem_levels(ix, &sbytes, cap);
    }
    p.Ls = Ls;
    p.smem_bytes = sbytes;
    p.stream_hint = (L.cache_hints & BS_HINT_STREAM_EVICT_FIRST) ? 1 : 0;
    p.leaf_hint = (L.cache_hints & BS_HINT_LEAF_EVICT_FIRST) ? 1 : 0;
    p.sep_hint = (L.cache_hints & BS_HINT_SEP_EVICT_LAST) ? 1 : 0;
    {   // separator levels (top-first) whose cumulative bytes fit half the L2 keep evict_last
        // (BS_SEP_L2_FRAC: A/B knob for the fraction, not part of the ABI)
        static const double frac = [] {
            const char* v = getenv("BS_SEP_L2_FRAC");
            const double f = v ? atof(v) : 0.5;
            return f > 0.0 && f <= 1.0 ? f : 0.5;
        }();
        const uint64_t l2 = ix->l2_bytes ? (uint64_t)ix->l2_bytes : (126ull << 20);
        uint64_t cum = 0;
        uint32_t end = 0;
        while (end < ix->kL) {
            const uint64_t lb = ix->k_nodes[end] * ix->kW * ix->kb;
            if (cum + lb > (uint64_t)(l2 * frac)) break;
            cum += lb;
            ++end;
        }
        p.sep_last_end = end;
    }
    const uint32_t smem = sbytes + 16;
    ix->last_kary_smem = smem;
    bool uns = false;
    Grid g{stat ? 1u : 0u, L.ctas_per_sm, (uint32_t)ix->sm_count};
    const uint32_t cpl = C >= W ? C / W : 1;
    if (g1) {
        // hi-word plane of the image only (u64), or the u32 plane
        uint32_t Li = 0;
        if (stat && L.use_pinned && ix->d_img) {
            const uint64_t cap = smem_cap(ix, L.ctas_per_sm ? L.ctas_per_sm : 1) - 16;
            const uint64_t budget = ix->layout.pin_bytes;
            while (Li < ix->img_L && (uint64_t)ix->img_base[Li + 1] * 4 <= cap &&
                   (budget == 0xFFFFFFFFu || (uint64_t)ix->img_base[Li + 1] * 4 <= budget))
                ++Li;
        }
        p.Ls = Li;
        // tie fix-up (kary_g1.cuh): node maxima of level Li = a[min((c+1)*span, n) - 1]
        if (Li > 0) {
            uint64_t span = ix->kC;
            for (uint32_t l = Li; l < ix->kL; ++l) span *= ix->kK;
            p.flat_span = span;
            p.flat_M = ix->k_next[Li - 1] - 1;
        }
        p.img = (const uint32_t*)ix->d_img;
        p.img_plane_words = ix->img_base[ix->img_L];
        for (uint32_t l = 0; l < Li; ++l) p.img_base[l] = ix->img_base[l];
        p.img_words = ix->img_base[Li];
        p.smem_bytes = p.img_words * 4 + 16;
        const bool flat = L.kary_mode == 7 && ix->d_flat && stat && L.use_pinned &&
                          (4ull << ix->flat_D) + 16 <= smem_cap(ix, L.ctas_per_sm ? L.ctas_per_sm : 1);
        if (flat) {
            p.Ls = ix->flat_level;
            p.flat = (const uint32_t*)ix->d_flat;
            p.flat64 = (const uint64_t*)ix->d_flat64;
            p.flat_D = ix->flat_D;
            p.flat_M = ix->flat_M;
            p.flat_span = ix->flat_span;
            p.fbase = ix->flat_fbase;
            p.fshift = ix->flat_fshift;
            p.smem_bytes = (4u << ix->flat_D) + 16;
            p.flat_img_words = 0;
            const uint64_t with_img = ((1ull << ix->flat_D) + ix->flat_img_words) * 4 + 16;
            // (not for the pipelined FLAT kernel, T = 3, which stages the table alone)
            const bool pipelined = (L.nreg >> 4) >= 3 && !pl;
            if (ix->d_flatimg && !pipelined && with_img <= smem_cap(ix, L.ctas_per_sm ? L.ctas_per_sm : 1)) {
                // table + the flat level's node image: one shared level more
                const uint32_t fl = ix->flat_level;
                p.Ls = fl + 1;
                p.flat = (const uint32_t*)ix->d_flatimg;
                p.flat_img_words = ix->flat_img_words;
                p.smem_bytes = (uint32_t)with_img;
                uint64_t span = ix->kC;
                for (uint32_t l = fl + 1; l < ix->kL; ++l) span *= ix->kK;
                p.flat_span = span;                 // tie fix-up at level fl + 1
                p.flat_M = ix->k_next[fl] - 1;
            }
        }
        ix->last_kary_smem = p.smem_bytes;
        // nreg: low 4 bits = leaf waves in flight IL (default 4), bits 4.. = lookups
        // per thread T (1 or 2, default 1)
        const uint32_t IL = (L.nreg & 15) ? (L.nreg & 15) : 4;
        uint32_t T = (L.nreg >> 4) ? (L.nreg >> 4) : 1;
        if (pl) T = 1;   // the peer epilogue is instantiated for one lookup per thread
        // T = 2 carries two lookups per thread in 80 registers: at most 768 threads
        // (T = 3 is the pipelined FLAT kernel, 1024 threads; without FLAT it runs as T = 2)
        const bool two = T == 2 || (T >= 3 && !flat);
        const uint32_t g1_threads = (two && !L.threads) ? 768u : threads;
        cudaError_t e = launch_kary_g1(ix->kb, ix->ob, &p, q, m, out, g1_threads, W, GL, IL, T, flat, g, p.smem_bytes, s, &uns);
        if (uns) return fail(BS_ERR_UNSUPPORTED, "KARY g1: threads=%u T=%u W=%u C=%u not supported", g1_threads, T, W, C);
        if (e != cudaSuccess) return fail_cuda(e, "KARY g1 launch");
        return BS_OK;
    }
    if (tiered) {
        // tiered: nreg = waves in flight (default 4, clamped to a divisor of the group size);
        // shared memory holds the image levels (odd node stride, hi/lo planes)
        const uint32_t I = L.nreg ? L.nreg : 4;
        // pair64: one plane of 8-B slots; else u64: hi/lo 4-B planes, u32: one 4-B plane
        const uint32_t planes = pair64 ? 1 : ix->kb == 8 ? 2 : 1;
        const uint32_t unit = pair64 ? 8 : 4;
        const uint32_t* base = pair64 ? ix->img64_base : ix->img_base;
        const uint32_t imgL = pair64 ? ix->img64_L : ix->img_L;
        const void* img = pair64 ? ix->d_img64 : ix->d_img;
        uint32_t Li = 0;
        if (stat && L.use_pinned && img) {
            const uint64_t cap = smem_cap(ix, L.ctas_per_sm ? L.ctas_per_sm : 1) - 16;
            const uint64_t budget = ix->layout.pin_bytes;   // image bytes (all planes)
            auto need = [&](uint64_t w) { return planes == 2 ? (29056ull + w) * 4 : w * unit; };
            while (Li < imgL && need(base[Li + 1]) <= cap &&
                   (budget == 0xFFFFFFFFu || (uint64_t)base[Li + 1] * unit * planes <= budget))
                ++Li;
        }
        p.Ls = Li;
        p.img = (const uint32_t*)img;
        p.img_plane_words = base[imgL];
        for (uint32_t l = 0; l < Li; ++l) p.img_base[l] = base[l];
        p.img_words = base[Li];   // units: 4-B words (planes) or 8-B slots (pair64)
        // smem: [hi plane | pad to the lo offset | lo plane | mbarrier] (u32 / pair64: [plane | mbarrier])
        p.smem_bytes = (Li == 0 ? 0u : planes == 2 ? (29056u + p.img_words) * 4 : p.img_words * unit) + 16;
        const uint32_t tsmem = p.smem_bytes;
        ix->last_kary_smem = tsmem;
        cudaError_t e = launch_kary_tiered(ix->kb, ix->ob, &p, q, m, out, threads, W, C / W, I, pair64, pipe, g, tsmem, s, &uns);
        if (uns) return fail(BS_ERR_UNSUPPORTED, "KARY tiered: threads=%u W=%u C=%u not supported", threads, W, C);
        if (e != cudaSuccess) return fail_cuda(e, "KARY tiered launch");
        return BS_OK;
    }
    if (L.kary_mode >= 1 && W <= 16 && cpl <= 4) {
        // hybrid: nreg = waves in flight (a divisor of W); default all W waves (32 lookups / warp)
        uint32_t I = L.nreg ? L.nreg : (W < 8 ? W : 8);
        if (I > W) I = W;
        cudaError_t e = launch_kary_hybrid(ix->kb, ix->ob, &p, q, m, out, threads, W, I, cpl, g, smem, s, &uns);
        if (uns) return fail(BS_ERR_UNSUPPORTED, "KARY hybrid: threads=%u waves=%u W=%u C=%u not supported", threads, I, W, C);
        if (e != cudaSuccess) return fail_cuda(e, "KARY hybrid launch");
        return BS_OK;
    }
    cudaError_t e = launch_kary(ix->kb, ix->ob, &p, q, m, out, threads, ix->kW, R, g, smem, s, &uns);
    if (uns) return fail(BS_ERR_UNSUPPORTED, "KARY: threads=%u waves=%u W=%u not supported", threads, R, ix->kW);
    if (e != cudaSuccess) return fail_cuda(e, "KARY launch");
    return BS_OK;
}

bool g1_shape_ok(const Index* ix) {
    const uint32_t W = ix->kW, C = ix->kC, kb = ix->kb;
    return ix->kary_built && (ix->layout.kary_mode == 6 || ix->layout.kary_mode == 7) && W * kb <= 64 &&
           W * kb >= 8 && C * kb >= 32 && C * kb <= 256;
}

int dispatch_kary_peer(const Index* ix, const void* q, uint64_t cap, cudaStream_t s, const bs_launch& L,
                       const PeerLaunch& pl) {
    if (L.variant != BS_VARIANT_KARY) return fail(BS_ERR_UNSUPPORTED, "bs_lookup_peer: needs variant KARY");
    return ix->kb == 8 ? run_kary<uint64_t>(ix, q, cap, nullptr, s, L, &pl)
                       : run_kary<uint32_t>(ix, q, cap, nullptr, s, L, &pl);
}

int dispatch_lookup(const Index* ix, const void* q, uint64_t m, void* out, cudaStream_t s, const bs_launch& L) {
    if (L.reorder == BS_REORDER_SORTED) {
        // an ordered batch (Fig. 1b): segment-staged lookup, any variant's index
        bool uns = false;
        Grid g{1u, 1u, (uint32_t)ix->sm_count};
        cudaError_t e = launch_seg_sorted(ix->kb, ix->ob, ix->d_keys, ix->n, q, m, out,
                                          (L.cache_hints & BS_HINT_STREAM_EVICT_FIRST) ? 1u : 0u, g, s, &uns);
        if (uns) return fail(BS_ERR_UNSUPPORTED, "BS_REORDER_SORTED: index too large for the segment table");
        if (e != cudaSuccess) return fail_cuda(e, "segment lookup launch");
        return BS_OK;
    }
    switch (L.variant) {
        case BS_VARIANT_NAIVE: {
            cudaError_t e = launch_naive(ix->kb, ix->ob, ix->d_keys, ix->n, q, m, out, L.threads, s);
            if (e != cudaSuccess) return fail_cuda(e, "NAIVE launch");
            return BS_OK;
        }
        case BS_VARIANT_OPT:
            return ix->kb == 8 ? run_opt<uint64_t>(ix, q, m, out, s, L) : run_opt<uint32_t>(ix, q, m, out, s, L);
        case BS_VARIANT_KARY:
            return ix->kb == 8 ? run_kary<uint64_t>(ix, q, m, out, s, L) : run_kary<uint32_t>(ix, q, m, out, s, L);
        default:
            return fail(BS_ERR_INVALID, "unknown variant %u", L.variant);
    }
}

}  // namespace bs
