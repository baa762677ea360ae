"""GPU parity of the ordered-batch path (BS_REORDER_SORTED, csrc/seg.cu) vs the
CPU oracle, bit-exact: sorted and unsorted batches (the latter exercise the
out-of-range fallback), u32/u64 keys, both output widths, segment-edge sizes,
duplicate runs straddling segment boundaries, keys that share their high word
(exact 32-bit image, sh = 0) and clustered keys in a wide span (many equal
images: the galloping fix-up)."""
import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402
from test_gpu_parity import build, check, run  # noqa: E402

S = 8192   # keys per segment (seg.cu kSegLog2)


def seg_run(idx, q, ob):
    return run(idx, q, ob, reorder=bs.REORDER_SORTED)


@pytest.fixture(params=["eytz", "bracket"])
def seg_kernel(request, monkeypatch):
    """Both SORTED kernels (seg.cu picks by queries per key; BS_SEG_KERNEL forces
    one): the image-tree descent and the bracketed bisection."""
    monkeypatch.setenv("BS_SEG_KERNEL", request.param)
    return request.param


def queries_for(keys, m, seed, order):
    q = workload.gen_queries(keys, m, seed=seed, hit_ratio=0.7)
    adv = workload.adversarial_queries(keys[:: max(1, keys.size // 500)], seed=seed, extra=300)
    q = np.concatenate([q, adv]).astype(keys.dtype)
    return np.sort(q) if order == "sorted" else q


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("order", ["sorted", "random"])
def test_seg_edge_sizes(kb, order, seg_kernel):
    for t, n in enumerate([1, 2, 3, 100, S - 1, S, S + 1, 2 * S, 3 * S + 5, 100003]):
        keys = workload.gen_keys(n, kb, seed=300 + t)
        q = queries_for(keys, 20000, 400 + t, order)
        for variant in (bs.NAIVE, bs.KARY):
            for ob in ((4, 8) if kb == 4 else (8,)):
                idx = build(keys, variant=variant, out_bytes=ob)
                check(seg_run(idx, q, ob), oracle.lookup(keys, q, out_bytes=ob), q, f"n={n} kb={kb} {order} ob={ob}")
                idx.close()


@pytest.mark.parametrize("kind", ["dups", "narrow", "clustered", "top"])
def test_seg_key_distributions(kind, seg_kernel):
    rng = np.random.default_rng({"dups": 1, "narrow": 2, "clustered": 3, "top": 4}[kind])
    n = 5 * S + 77
    if kind == "dups":
        # runs of equal keys, some spanning whole segments, straddling every boundary
        v = np.repeat(rng.integers(0, 1 << 62, size=n // 40, dtype=np.uint64), 40)
        v = np.concatenate([v, np.full(2 * S + 3, 1 << 61, dtype=np.uint64)])
    elif kind == "narrow":
        v = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)              # every key < 2^32
    elif kind == "clustered":
        v = np.concatenate([rng.integers(0, 1 << 20, size=n // 2, dtype=np.uint64),
                            rng.integers(0, 1 << 63, size=n // 2, dtype=np.uint64) * np.uint64(2)])
    else:
        v = np.concatenate([np.full(S + 9, (1 << 64) - 1, dtype=np.uint64),
                            rng.integers((1 << 64) - (1 << 40), (1 << 64) - 1, size=n, dtype=np.uint64)])
    keys = np.sort(v)
    for order in ("sorted", "random"):
        q = queries_for(keys, 50000, 7, order)
        idx = build(keys, variant=bs.KARY, out_bytes=8)
        check(seg_run(idx, q, 8), oracle.lookup(keys, q, out_bytes=8), q, f"{kind} {order}")
        idx.close()


def test_seg_config3_sorted_sample(seg_kernel):
    """BASELINE configs[2] keys, pre-sorted 2^24-query batch: sampled oracle + every output's invariant."""
    import bench
    dk, dq, _ = bench._gen("config3", 0, 1, "strong", "sorted", "cuda")
    dq = dq[: 1 << 24].contiguous()      # a prefix of a sorted batch is sorted
    m = dq.numel()
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    idx = bs.bs_build(dk, dk.numel(), bs.bs_layout_default())
    bs.bs_lookup_ex(idx, dq, m, out, None, reorder=bs.REORDER_SORTED)
    torch.cuda.synchronize()
    kh, qh = bench._host(dk, 8), bench._host(dq, 8)
    samp = np.random.default_rng(5).integers(0, m, size=1 << 15)
    assert np.array_equal(P.to_numpy_unsigned(out, 8)[samp], oracle.lookup(kh, qh[samp], out_bytes=8))
    assert bench.invariant_all(dk, dq, out, 8)
    idx.close()


# ------------------------------------------------------------------ BS_REORDER_GLOBAL (partition -> segments -> unpartition)

def glob_run(idx, q, ob):
    dq = P.as_torch(q)
    out = torch.full((max(q.size, 1),), -1, dtype={4: torch.int32, 8: torch.int64}[ob], device="cuda")
    nb = bs.bs_workspace_bytes(idx, q.size, reorder=bs.REORDER_GLOBAL)
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")
    bs.bs_lookup_ws(idx, dq, q.size, out, None, ws, nb, reorder=bs.REORDER_GLOBAL)
    torch.cuda.synchronize()
    return P.to_numpy_unsigned(out, ob)[: q.size]


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("order", ["random", "sorted"])
def test_global_edge_sizes(kb, order):
    SG = 32768   # GLOBAL mode bucket segment (seg.cu kGlobLog2)
    for t, n in enumerate([1, 2, 100, S + 1, SG - 1, SG, SG + 1, 3 * SG + 5, 300007]):
        keys = workload.gen_keys(n, kb, seed=500 + t)
        for m in (1, 777, 8191, 8192, 8193, 30011):
            q = queries_for(keys, m, 600 + t, order)
            for ob in ((4, 8) if kb == 4 else (8,)):
                idx = build(keys, variant=bs.KARY, out_bytes=ob)
                check(glob_run(idx, q, ob), oracle.lookup(keys, q, out_bytes=ob), q, f"n={n} m={q.size} kb={kb} {order} ob={ob}")
                idx.close()


@pytest.mark.parametrize("kind", ["dups", "narrow", "clustered", "top"])
def test_global_key_distributions(kind):
    rng = np.random.default_rng({"dups": 11, "narrow": 12, "clustered": 13, "top": 14}[kind])
    SG = 32768
    n = 5 * SG + 77
    if kind == "dups":
        v = np.repeat(rng.integers(0, 1 << 62, size=n // 40, dtype=np.uint64), 40)
        v = np.concatenate([v, np.full(2 * SG + 3, 1 << 61, dtype=np.uint64)])
    elif kind == "narrow":
        v = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
    elif kind == "clustered":
        v = np.concatenate([rng.integers(0, 1 << 20, size=n // 2, dtype=np.uint64),
                            rng.integers(0, 1 << 63, size=n // 2, dtype=np.uint64) * np.uint64(2)])
    else:
        v = np.concatenate([np.full(SG + 9, (1 << 64) - 1, dtype=np.uint64),
                            rng.integers((1 << 64) - (1 << 40), (1 << 64) - 1, size=n, dtype=np.uint64)])
    keys = np.sort(v)
    q = queries_for(keys, 200000, 8, "random")
    idx = build(keys, variant=bs.KARY, out_bytes=8)
    check(glob_run(idx, q, 8), oracle.lookup(keys, q, out_bytes=8), q, kind)
    idx.close()


def test_global_skewed_batch_overflows():
    """Every query in one segment: its region overflows (cap = 1.25 m/B + 64) and
    the overflow list is looked up by global bisection — same results."""
    keys = workload.gen_keys(6 * 32768, 8, seed=21)
    hot = keys[2 * 32768: 2 * 32768 + 50]
    rng = np.random.default_rng(3)
    q = np.concatenate([rng.choice(hot, 40000), workload.gen_queries(keys, 5000, seed=4)])
    q = q[rng.permutation(q.size)]
    idx = build(keys, variant=bs.KARY, out_bytes=8)
    check(glob_run(idx, q, 8), oracle.lookup(keys, q, out_bytes=8), q, "skewed")
    idx.close()


def test_global_needs_workspace():
    keys = workload.gen_keys(1000, 8, seed=1)
    idx = build(keys, variant=bs.KARY)
    dq = P.as_torch(keys)
    out = torch.empty(keys.size, dtype=torch.int64, device="cuda")
    with pytest.raises(bs.BsError) as e:
        bs.bs_lookup_ex(idx, dq, keys.size, out, None, reorder=bs.REORDER_GLOBAL)
    assert e.value.code == bs.BS_ERR_INVALID
    nb = bs.bs_workspace_bytes(idx, keys.size, reorder=bs.REORDER_GLOBAL)
    ws = torch.empty(nb - 256, dtype=torch.uint8, device="cuda")
    with pytest.raises(bs.BsError) as e:
        bs.bs_lookup_ws(idx, dq, keys.size, out, None, ws, nb - 256, reorder=bs.REORDER_GLOBAL)
    assert e.value.code == bs.BS_ERR_INVALID
    assert bs.bs_workspace_bytes(idx, keys.size) == 0       # the default mode needs none
    idx.close()


def test_global_config3_sample():
    """BASELINE configs[2] (2^26 u64 keys, 2^27 random queries), GLOBAL mode: sampled oracle + every output's invariant."""
    import bench
    dk, dq, _ = bench._gen("config3", 0, 1, "strong", "random", "cuda")
    m = dq.numel()
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    idx = bs.bs_build(dk, dk.numel(), bs.bs_layout_default())
    nb = bs.bs_workspace_bytes(idx, m, reorder=bs.REORDER_GLOBAL)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    bs.bs_lookup_ws(idx, dq, m, out, None, ws, nb, reorder=bs.REORDER_GLOBAL)
    torch.cuda.synchronize()
    kh, qh = bench._host(dk, 8), bench._host(dq, 8)
    samp = np.random.default_rng(6).integers(0, m, size=1 << 15)
    assert np.array_equal(P.to_numpy_unsigned(out, 8)[samp], oracle.lookup(kh, qh[samp], out_bytes=8))
    assert bench.invariant_all(dk, dq, out, 8)
    idx.close()
