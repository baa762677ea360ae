"""GPU parity: every variant and knob of libbs.so vs the CPU oracle, bit-exact.

Inputs come from workload/ (seeded); expected values from oracle/ only.
All calls go through the C ABI (paper_2506_01576_b200.bs).
"""
import itertools

import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402

ODT = {4: torch.int32, 8: torch.int64}


def run(idx, q_np, out_bytes, **launch):
    dq = P.as_torch(q_np)
    out = torch.full((max(q_np.size, 1),), -1, dtype=ODT[out_bytes], device="cuda")
    if launch:
        bs.bs_lookup_ex(idx, dq, q_np.size, out, **launch)
    else:
        bs.bs_lookup(idx, dq, q_np.size, out)
    torch.cuda.synchronize()
    return P.to_numpy_unsigned(out, out_bytes)[: q_np.size]


def check(got, want, q, tag=""):
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)
        i = int(bad[0])
        raise AssertionError(f"{tag}: {bad.size} mismatches; first at {i}: q={int(q[i]):#x} "
                             f"got={int(got[i]):#x} want={int(want[i]):#x}")


def build(keys, **kw):
    kb = keys.dtype.itemsize
    lay = bs.bs_layout_default(key_bytes=kb, out_bytes=kw.pop("out_bytes", kb), **kw)
    return bs.bs_build(P.as_torch(keys), keys.size, lay)


# ------------------------------------------------------------------ config 1

@pytest.mark.parametrize("variant", [bs.NAIVE, bs.OPT, bs.KARY])
@pytest.mark.parametrize("out_bytes", [4, 8])
def test_config1(variant, out_bytes):
    """BASELINE.json configs[0]: 2^10 u32 keys, 2^16 queries, 50 % hits."""
    keys = workload.gen_keys(1 << 10, 4)
    q = workload.gen_queries(keys, 1 << 16, hit_ratio=0.5)
    want = oracle.lookup(keys, q, out_bytes=out_bytes)
    idx = build(keys, variant=variant, out_bytes=out_bytes)
    check(run(idx, q, out_bytes), want, q, f"variant {variant}")


# ------------------------------------------------------------------ edge sizes

EDGE_N = [1, 2, 3, 4, 5, 7, 8, 9, 14, 15, 16, 17, 27, 31, 32, 33, 63, 64, 65, 255, 256, 257,
          1000, 1023, 1024, 1025, 4095, 4096, 4097, 12345, 65535, 65536, 65537]


def edge_keys(n, kb, seed):
    dt = workload.key_dtype(kb)
    if n <= 64 or seed % 3 == 0:
        # dense small domain with duplicates and MAX at the end
        rng = np.random.default_rng(seed)
        v = np.sort(rng.integers(0, 3 * n + 2, size=n).astype(dt))
        if seed % 2:
            v[-1] = np.iinfo(dt).max
        return v
    return workload.gen_keys(n, kb, seed=seed)


@pytest.mark.parametrize("kb", [4, 8])
def test_edge_sizes_all_variants(kb):
    for t, n in enumerate(EDGE_N):
        keys = edge_keys(n, kb, seed=100 + t)
        q = workload.adversarial_queries(keys, seed=t, extra=200)
        want = oracle.lookup(keys, q)
        for variant in (bs.NAIVE, bs.OPT, bs.KARY):
            idx = build(keys, variant=variant)
            check(run(idx, q, kb), want, q, f"n={n} kb={kb} variant={variant}")
            idx.close()


# ------------------------------------------------------------------ OPT knobs

def opt_grid():
    full = []
    for threads, nreg in itertools.product([64, 128, 256, 512, 1024], [1, 2, 4, 8, 16]):
        for reorder in (0, 1, 2):
            full.append(dict(threads=threads, nreg=nreg, reorder=reorder))
    return full


@pytest.mark.parametrize("kb", [4, 8])
def test_opt_knob_cross_product(kb):
    """threads x NREG x reorder x {pinned full / steps / none} x {static / dynamic};
    unsupported combinations (register / shared-memory limits) must say so."""
    n = 100003
    keys = workload.gen_keys(n, kb, seed=5)
    q = workload.gen_queries(keys, 300007, seed=6, hit_ratio=0.7)
    want = oracle.lookup(keys, q)
    idx = build(keys, variant=bs.OPT)
    ran = 0
    for cfg in opt_grid():
        for use_pinned, partial in ((1, 1), (1, 0), (0, 0)):
            for sched in (bs.STATIC, bs.DYNAMIC):
                try:
                    got = run(idx, q, kb, variant=bs.OPT, schedule=sched, use_pinned=use_pinned,
                              pin_partial=partial, **cfg)
                except bs.BsError as e:
                    assert e.code == bs.BS_ERR_UNSUPPORTED, str(e)
                    continue
                check(got, want, q, f"{cfg} pinned={use_pinned} partial={partial} sched={sched}")
                ran += 1
    assert ran > 150


@pytest.mark.parametrize("pin_bytes", [16, 48, 1024, 40000, 0xFFFFFFFF])
def test_opt_pin_budgets(pin_bytes):
    """Budgets from one entry to the largest table (levels complete / partial / whole array)."""
    for n in (2, 14, 1000, 4096, 5000, 1 << 20):
        keys = edge_keys(n, 8, seed=n)
        q = workload.adversarial_queries(keys, seed=n, extra=3000)
        want = oracle.lookup(keys, q)
        idx = build(keys, variant=bs.OPT, pin_bytes=pin_bytes)
        for partial in (0, 1):
            check(run(idx, q, 8, pin_partial=partial, use_pinned=1), want, q, f"n={n} pin={pin_bytes} p={partial}")


# ------------------------------------------------------------------ K-ary knobs

@pytest.mark.parametrize("kb", [4, 8])
def test_kary_k_c_waves(kb):
    """K in {2..33} x C in {1..64} x waves {1,2,4,8} x smem levels on/off x schedule."""
    n = 77777
    keys = edge_keys(n, kb, seed=9)
    q = workload.adversarial_queries(keys, seed=9, extra=5000)[:60000]
    want = oracle.lookup(keys, q)
    for K in (2, 3, 4, 5, 8, 9, 16, 17, 32, 33):
        for C in (1, 2, 4, 8, 16, 32, 64):
            idx = build(keys, variant=bs.KARY, k=K, leaf_chunk=C)
            for mode in (7, 6, 5, 4, 3, 2, 1, 0):
                for R, sched, pin in ((1, bs.STATIC, 1), (2, bs.DYNAMIC, 0), (4, bs.STATIC, 0), (8, bs.STATIC, 1)):
                    got = run(idx, q, kb, variant=bs.KARY, nreg=R, schedule=sched, use_pinned=pin,
                              threads=256 if R < 8 else 128, kary_mode=mode)
                    check(got, want, q, f"K={K} C={C} R={R} sched={sched} pin={pin} mode={mode}")
            idx.close()


@pytest.mark.parametrize("kb,ob", [(8, 8), (8, 4), (4, 4), (4, 8)])
def test_kary_tiered_out_widths(kb, ob):
    """Tiered schedule (kary_mode 2): both key widths x both result widths, hits and misses."""
    keys = edge_keys(100003, kb, seed=21)
    q = workload.adversarial_queries(keys, seed=21, extra=20000)
    want = oracle.lookup(keys, q, out_bytes=ob)
    for K, C in ((17, 16), (16, 16), (9, 16), (5, 8), (33, 32), (3, 4), (9, 32), (5, 16), (4, 16), (3, 16), (8, 32)):
        idx = build(keys, variant=bs.KARY, k=K, leaf_chunk=C, out_bytes=ob)
        for mode in (2, 3, 4, 5, 6, 7):
            for I in (1, 2, 4) if mode < 6 else (1, 2, 4, 0x24, 0x34):   # g1: T=2 / pipelined (T=3)
                check(run(idx, q, ob, kary_mode=mode, nreg=I), want, q, f"tiered{mode} K={K} C={C} I={I} kb={kb} ob={ob}")
        idx.close()


def test_kary_small_n_all_shapes():
    for n in (1, 2, 3, 5, 16, 17, 33, 100):
        for K in (2, 3, 17, 33):
            for C in (1, 4, 32):
                keys = edge_keys(n, 8, seed=n * 7 + K)
                q = workload.adversarial_queries(keys, seed=K, extra=50)
                idx = build(keys, variant=bs.KARY, k=K, leaf_chunk=C)
                for mode in (7, 6, 5, 4, 3, 2, 1, 0):
                    check(run(idx, q, 8, kary_mode=mode), oracle.lookup(keys, q), q, f"n={n} K={K} C={C} mode={mode}")


# ------------------------------------------------------------------ misc semantics

def test_m_edge_cases():
    keys = workload.gen_keys(5000, 8, seed=1)
    for variant in (bs.NAIVE, bs.OPT, bs.KARY):
        idx = build(keys, variant=variant)
        for m in (0, 1, 31, 2047, 2048, 2049, 4097):
            q = workload.gen_queries(keys, m, seed=m, hit_ratio=0.5)
            if m == 0:
                out = torch.empty(1, dtype=torch.int64, device="cuda")
                bs.bs_lookup(idx, P.as_torch(np.zeros(1, np.uint64)), 0, out)
                continue
            check(run(idx, q, 8), oracle.lookup(keys, q), q, f"m={m} variant={variant}")


def test_unsorted_input_is_sorted_by_library():
    """input_sorted = 0: the library sorts a copy with unsigned order (keys >= 2^63, duplicates)."""
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 2**64 - 1, size=50000, dtype=np.uint64, endpoint=True)
    keys[:1000] = keys[1000:2000]   # duplicates
    q = workload.adversarial_queries(np.sort(keys), seed=2, extra=1000)
    want = oracle.lookup(np.sort(keys), q)
    for variant in (bs.NAIVE, bs.OPT, bs.KARY):
        idx = build(keys, variant=variant, input_sorted=0)
        check(run(idx, q, 8), want, q, f"unsorted variant={variant}")
        assert np.array_equal(bs.bs_export(idx, bs.EXPORT_SORTED), np.sort(keys))


def test_not_sorted_rejected():
    keys = np.array([3, 1, 2], dtype=np.uint64)
    with pytest.raises(bs.BsError) as e:
        build(keys, variant=bs.KARY, input_sorted=1)
    assert e.value.code == bs.BS_ERR_NOT_SORTED


def test_overlap_rejected():
    keys = workload.gen_keys(100, 8, seed=1)
    idx = build(keys)
    buf = torch.zeros(64, dtype=torch.int64, device="cuda")
    with pytest.raises(bs.BsError) as e:
        bs.bs_lookup(idx, buf, 32, buf[16:])
    assert e.value.code == bs.BS_ERR_INVALID


def test_sorted_and_random_order_config3_small():
    """Fig. 1b workload shape at a small size: random vs pre-sorted queries."""
    keys = workload.gen_keys(1 << 20, 8)
    for order in ("random", "sorted"):
        q = workload.gen_queries(keys, 1 << 21, order=order)
        want = oracle.lookup(keys, q, threads=8)
        for variant in (bs.NAIVE, bs.OPT, bs.KARY):
            idx = build(keys, variant=variant)
            check(run(idx, q, 8), want, q, f"{order} variant={variant}")


def test_host_path_pinned_and_pageable():
    keys = workload.gen_keys(1 << 16, 8, seed=4)
    q = workload.gen_queries(keys, (1 << 23) + 12345, seed=5, hit_ratio=0.9)
    want = oracle.lookup(keys, q, threads=8)
    idx = build(keys)
    out = np.empty(q.size, dtype=np.uint64)
    bs.bs_lookup_host(idx, q, q.size, out)     # pageable numpy buffers
    check(out, want, q, "host pageable")
    tq = torch.from_numpy(q.view(np.int64)).pin_memory()
    to = torch.empty(q.size, dtype=torch.int64).pin_memory()
    bs.bs_lookup_host(idx, tq, q.size, to)
    check(to.numpy().view(np.uint64), want, q, "host pinned")


def test_info_footprint():
    keys = workload.gen_keys(1 << 20, 4)
    idx = build(keys, variant=bs.KARY, k=17, leaf_chunk=32)
    info = idx.info
    assert info["n"] == 1 << 20 and info["array_bytes"] == 4 << 20
    # separators: 2^20 / 32 chunks, K = 17 -> 32800 real separators (P:252 ~3.1 %)
    assert info["kary_levels"] == 4
    assert info["separator_bytes"] >= 32800 * 4
    assert info["footprint_bytes"] >= info["array_bytes"] + info["separator_bytes"]
    assert info["build_ms"] > 0


# ------------------------------------------------------------------ u64 keys in a narrow range (hi-word ties)

@pytest.mark.parametrize("hi_log2", [20, 32, 40, 48])
def test_u64_narrow_key_range(hi_log2):
    """u64 keys confined to [0, 2^hi): with the high word alone every probe of the
    flat table would tie; the order-preserving image (span in 32 bits) and the
    galloping fix-up must give the oracle's results for every schedule."""
    from workload import device as wd
    n = min(1 << 20, (1 << hi_log2) // 4)
    keys = wd.gen_keys_range(n, 0, 1 << hi_log2, 77, 0, device="cpu").numpy().view(np.uint64)
    q = np.concatenate([workload.gen_queries(keys, 200000, seed=3, hit_ratio=0.8),
                        workload.adversarial_queries(keys[::97], seed=5, extra=500)])
    want = oracle.lookup(keys, q)
    idx = build(keys, variant=bs.KARY)
    check(run(idx, q, 8), want, q, f"default hi={hi_log2}")
    for mode in (6, 7):
        check(run(idx, q, 8, kary_mode=mode), want, q, f"mode {mode} hi={hi_log2}")
    check(run(idx, q, 8, kary_mode=7, nreg=0x34), want, q, f"pipelined hi={hi_log2}")
    idx.close()


# ------------------------------------------------------------------ boundary (§8b error table)

def test_lookup_rejects_host_pointers():
    """bs_lookup takes device memory only (P:61 'all data GPU-resident'); a host
    buffer is BS_ERR_INVALID, not an asynchronous fault (host buffers: bs_lookup_host)."""
    keys = workload.gen_keys(5000, 8, seed=2)
    q = workload.gen_queries(keys, 1000, seed=3)
    idx = build(keys, variant=bs.KARY)
    dq = P.as_torch(q)
    out = torch.empty(q.size, dtype=torch.int64, device="cuda")
    hq = torch.from_numpy(q.view(np.int64))
    hout = torch.empty(q.size, dtype=torch.int64)
    for a, b in ((hq, out), (dq, hout), (hq.pin_memory(), out), (dq, hout.pin_memory())):
        with pytest.raises(bs.BsError) as e:
            bs.bs_lookup(idx, a, q.size, b)
        assert e.value.code == bs.BS_ERR_INVALID
    bs.bs_lookup(idx, dq, q.size, out)          # the device path still works
    torch.cuda.synchronize()
    check(P.to_numpy_unsigned(out, 8), oracle.lookup(keys, q), q, "after rejections")
    idx.close()


def test_concurrent_lookups_on_streams():
    """An index is immutable: lookups on one index from many streams / host
    threads at once give the oracle's results (the launch-plan cache and the
    shared-memory statistics are the only shared mutable state)."""
    import threading
    keys = workload.gen_keys(1 << 20, 8, seed=4)
    idx = build(keys, variant=bs.KARY)
    qs = [workload.gen_queries(keys, 1 << 18, seed=10 + i, hit_ratio=0.7) for i in range(8)]
    dqs = [P.as_torch(q) for q in qs]
    outs = [torch.empty(q.size, dtype=torch.int64, device="cuda") for q in qs]
    streams = [torch.cuda.Stream() for _ in qs]
    launches = [dict(), dict(kary_mode=6), dict(variant=bs.OPT), dict(variant=bs.NAIVE),
                dict(reorder=bs.REORDER_SORTED), dict(kary_mode=7, nreg=0x24), dict(), dict(kary_mode=0)]
    errs = []

    def work(i):
        try:
            for _ in range(3):
                bs.bs_lookup_ex(idx, dqs[i], qs[i].size, outs[i], streams[i], **launches[i])
        except Exception as ex:   # pragma: no cover - reported below
            errs.append(ex)
    th = [threading.Thread(target=work, args=(i,)) for i in range(len(qs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for i, q in enumerate(qs):
        check(P.to_numpy_unsigned(outs[i], 8), oracle.lookup(keys, q), q, f"stream {i} {launches[i]}")
    idx.close()
