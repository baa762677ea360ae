"""GPU parity of the bucket-partitioned lookup (BS_REORDER_BUCKET, csrc/part.cu)
vs the CPU oracle, bit-exact: bucket-edge array sizes (a bucket = 2^15 leaves of
32 B: 2^17 u64 / 2^18 u32 keys), tile-edge batch sizes (4096-query partition
tiles), both orders, u32/u64 keys, both output widths, duplicate runs straddling
bucket edges, keys sharing their high word (exact images), clustered keys in a
wide span (equal images: the galloping fix-ups), MAX keys, a batch that falls
into one bucket, the workspace contract, and BASELINE configs[2] in full."""
import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402
from test_gpu_parity import build, check  # noqa: E402

NB = {8: 1 << 17, 4: 1 << 18}   # keys per bucket (part.cu: 2^15 leaves of 32 B)
T = 8192                          # queries per partition tile


def bk_run(idx, q, ob):
    dq = P.as_torch(q)
    out = torch.full((max(q.size, 1),), -1, dtype={4: torch.int32, 8: torch.int64}[ob], device="cuda")
    nb = bs.bs_workspace_bytes(idx, q.size, reorder=bs.REORDER_BUCKET)
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")
    bs.bs_lookup_ws(idx, dq, q.size, out, None, ws, nb, reorder=bs.REORDER_BUCKET)
    torch.cuda.synchronize()
    return P.to_numpy_unsigned(out, ob)[: q.size]


def queries_for(keys, m, seed, order, hit_ratio=0.7):
    q = workload.gen_queries(keys, m, seed=seed, hit_ratio=hit_ratio)
    adv = workload.adversarial_queries(keys[:: max(1, keys.size // 500)], seed=seed, extra=300)
    q = np.concatenate([q, adv]).astype(keys.dtype)
    return np.sort(q) if order == "sorted" else q


@pytest.mark.parametrize("kb", [4, 8])
def test_bucket_edge_sizes(kb):
    nb = NB[kb]
    for t, n in enumerate([1, 2, 3, 5, 100, nb - 1, nb, nb + 1, 2 * nb + 5, 3 * nb - 3]):
        keys = workload.gen_keys(n, kb, seed=700 + t)
        for m in (1, 31, T - 1, T + 1, 3 * T + 17):
            for order in ("random", "sorted"):
                q = queries_for(keys, m, 800 + t, order)
                for ob in ((4, 8) if kb == 4 else (8,)):
                    idx = build(keys, variant=bs.KARY, out_bytes=ob)
                    check(bk_run(idx, q, ob), oracle.lookup(keys, q, out_bytes=ob), q,
                          f"n={n} m={q.size} kb={kb} {order} ob={ob}")
                    idx.close()


@pytest.mark.parametrize("variant", [bs.NAIVE, bs.OPT])
def test_bucket_any_variant(variant):
    """The bucket tables are built for every variant's index."""
    keys = workload.gen_keys(3 * NB[8] + 11, 8, seed=31)
    q = queries_for(keys, 100000, 32, "random")
    idx = build(keys, variant=variant, out_bytes=8)
    check(bk_run(idx, q, 8), oracle.lookup(keys, q, out_bytes=8), q, f"variant {variant}")
    idx.close()


@pytest.mark.parametrize("kind", ["dups", "narrow", "narrow40", "clustered", "top", "bottom"])
def test_bucket_key_distributions(kind):
    rng = np.random.default_rng({"dups": 21, "narrow": 22, "narrow40": 23, "clustered": 24, "top": 25,
                                 "bottom": 26}[kind])
    nb = NB[8]
    n = 4 * nb + 77
    if kind == "dups":
        # runs of equal keys, some longer than a leaf / a bucket, straddling every bucket edge
        v = np.repeat(rng.integers(0, 1 << 62, size=n // 40, dtype=np.uint64), 40)
        v = np.concatenate([v, np.full(nb + 3, 1 << 61, dtype=np.uint64), np.full(37, 5, dtype=np.uint64)])
    elif kind == "narrow":
        v = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)              # every key < 2^32: exact images
    elif kind == "narrow40":
        v = rng.integers(0, 1 << 40, size=n, dtype=np.uint64)
    elif kind == "clustered":
        # half the keys in [0, 2^20), half spread over 2^64: equal images inside the straddling bucket
        v = np.concatenate([rng.integers(0, 1 << 20, size=n // 2, dtype=np.uint64),
                            rng.integers(0, 1 << 63, size=n // 2, dtype=np.uint64) * np.uint64(2)])
    elif kind == "top":
        v = np.concatenate([np.full(nb + 9, (1 << 64) - 1, dtype=np.uint64),
                            rng.integers((1 << 64) - (1 << 40), (1 << 64) - 1, size=n, dtype=np.uint64)])
    else:
        v = np.concatenate([np.zeros(nb // 2, dtype=np.uint64),
                            rng.integers(0, 1 << 64, size=n, dtype=np.uint64, endpoint=False)])
    keys = np.sort(v)
    for order in ("random", "sorted"):
        q = queries_for(keys, 200000, 9, order)
        idx = build(keys, variant=bs.KARY, out_bytes=8)
        check(bk_run(idx, q, 8), oracle.lookup(keys, q, out_bytes=8), q, f"{kind} {order}")
        idx.close()


def test_bucket_skewed_batch():
    """Every query of most tiles in one bucket (runs as long as a tile) plus empty buckets."""
    keys = workload.gen_keys(6 * NB[8], 8, seed=41)
    hot = keys[2 * NB[8]: 2 * NB[8] + 50]
    rng = np.random.default_rng(3)
    q = np.concatenate([rng.choice(hot, 40000), workload.gen_queries(keys, 5000, seed=4)])
    q = q[rng.permutation(q.size)]
    idx = build(keys, variant=bs.KARY, out_bytes=8)
    check(bk_run(idx, q, 8), oracle.lookup(keys, q, out_bytes=8), q, "skewed")
    idx.close()


def test_bucket_needs_workspace():
    keys = workload.gen_keys(1000, 8, seed=1)
    idx = build(keys, variant=bs.KARY)
    dq = P.as_torch(keys)
    out = torch.empty(keys.size, dtype=torch.int64, device="cuda")
    with pytest.raises(bs.BsError) as e:
        bs.bs_lookup_ex(idx, dq, keys.size, out, None, reorder=bs.REORDER_BUCKET)
    assert e.value.code == bs.BS_ERR_INVALID
    nb = bs.bs_workspace_bytes(idx, keys.size, reorder=bs.REORDER_BUCKET)
    ws = torch.empty(nb - 256, dtype=torch.uint8, device="cuda")
    with pytest.raises(bs.BsError) as e:
        bs.bs_lookup_ws(idx, dq, keys.size, out, None, ws, nb - 256, reorder=bs.REORDER_BUCKET)
    assert e.value.code == bs.BS_ERR_INVALID
    idx.close()


def test_bucket_config3_sample():
    """BASELINE configs[2] (2^26 u64 keys, 2^27 random queries), BUCKET mode: sampled oracle + every output's invariant."""
    import bench
    dk, dq, _ = bench._gen("config3", 0, 1, "strong", "random", "cuda")
    m = dq.numel()
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    idx = bs.bs_build(dk, dk.numel(), bs.bs_layout_default())
    nb = bs.bs_workspace_bytes(idx, m, reorder=bs.REORDER_BUCKET)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    bs.bs_lookup_ws(idx, dq, m, out, None, ws, nb, reorder=bs.REORDER_BUCKET)
    torch.cuda.synchronize()
    kh, qh = bench._host(dk, 8), bench._host(dq, 8)
    samp = np.random.default_rng(7).integers(0, m, size=1 << 15)
    assert np.array_equal(P.to_numpy_unsigned(out, 8)[samp], oracle.lookup(kh, qh[samp], out_bytes=8))
    assert bench.invariant_all(dk, dq, out, 8)
    idx.close()


@pytest.mark.timeout(900)
def test_bucket_max_batch():
    """The largest batch BUCKET mode takes (m < 2^32, ragged: 2^32 - 2^20 - 3
    u32 queries over 2^26 u32 keys, 256 fine buckets): bucket counts, run
    positions and the search's item ranges are 32-bit and wrap nowhere.  Checked
    on 2^16 sampled outputs and on the first and last 2^16 outputs."""
    import workload.device as wd
    free, _ = torch.cuda.mem_get_info()
    m = (1 << 32) - (1 << 20) - 3
    if free < 100 * (1 << 30):
        pytest.skip("needs ~100 GB of free device memory")
    dk = wd.gen_keys(1 << 26, 4, device="cuda")
    dq = wd.gen_queries(dk, m, hit_ratio=0.7)
    out = torch.empty(m, dtype=torch.int32, device="cuda")
    idx = bs.bs_build(dk, dk.numel(), bs.bs_layout_default(key_bytes=4, out_bytes=4))
    nb = bs.bs_workspace_bytes(idx, m, reorder=bs.REORDER_BUCKET)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    bs.bs_lookup_ws(idx, dq, m, out, None, ws, nb, reorder=bs.REORDER_BUCKET)
    torch.cuda.synchronize()
    kh = P.to_numpy_unsigned(dk, 4)
    samp = np.concatenate([np.arange(1 << 16), np.arange(m - (1 << 16), m),
                           np.random.default_rng(9).integers(0, m, size=1 << 16)])
    st = torch.from_numpy(samp).cuda()
    got = P.to_numpy_unsigned(out[st], 4)
    want = oracle.lookup(kh, P.to_numpy_unsigned(dq[st], 4), out_bytes=4)
    assert np.array_equal(got, want), f"first mismatch at {samp[np.flatnonzero(got != want)[:5]]}"
    idx.close()


# ------------------------------------------------------------------ two-level buckets (large arrays)

@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("variant", [bs.KARY, bs.OPT, bs.NAIVE])
def test_bucket_two_level(kb, variant, monkeypatch):
    """Two-level buckets (2^15 units of 16 leaves of 32 B with a 32-B node of 16-bit
    leaf-maxima images relative to the unit; the A/B knob BS_BUCKET_G8=1: units of
    8 leaves of 64 B with 32-bit node images) — the layout bs_build picks above 2^27 u64 / 2^28 u32 keys;
    forced here with BS_BUCKET_TWO=1 on arrays of a few buckets.  Also the A/B
    path that searches the partitioned batch with the index's own kernel
    (BS_BUCKET_KARY=1)."""
    monkeypatch.setenv("BS_BUCKET_TWO", "1")
    per = (16 << 20) // kb
    n = 2 * per + 12345
    keys = workload.gen_keys(n, kb, seed=900 + kb + variant)
    for order in ("random", "sorted"):
        q = queries_for(keys, 150000, 901, order)
        for ob in ((4, 8) if kb == 4 else (8,)):
            want = oracle.lookup(keys, q, out_bytes=ob)
            for g8 in ("0", "1"):
                monkeypatch.setenv("BS_BUCKET_G8", g8)
                idx = build(keys, variant=variant, out_bytes=ob)
                check(bk_run(idx, q, ob), want, q, f"two-level kb={kb} v={variant} {order} ob={ob} g8={g8}")
                monkeypatch.setenv("BS_BUCKET_KARY", "1")
                check(bk_run(idx, q, ob), want, q, f"partitioned own-kernel kb={kb} v={variant} {order} ob={ob}")
                monkeypatch.delenv("BS_BUCKET_KARY")
                idx.close()


@pytest.mark.parametrize("kind", ["dups", "clustered", "top"])
def test_bucket_two_level_distributions(kind, monkeypatch):
    """Image ties at the node level (clustered keys in a wide span), duplicate
    runs across leaves / units / buckets, MAX keys — two-level buckets."""
    monkeypatch.setenv("BS_BUCKET_TWO", "1")
    rng = np.random.default_rng({"dups": 31, "clustered": 32, "top": 33}[kind])
    per = 1 << 21
    n = 2 * per + 777
    if kind == "dups":
        v = np.repeat(rng.integers(0, 1 << 62, size=n // 100, dtype=np.uint64), 100)
        v = np.concatenate([v, np.full(per + 5, 1 << 61, dtype=np.uint64)])
    elif kind == "clustered":
        v = np.concatenate([rng.integers(0, 1 << 16, size=n // 2, dtype=np.uint64),
                            rng.integers(0, 1 << 63, size=n // 2, dtype=np.uint64) * np.uint64(2)])
    else:
        v = np.concatenate([np.full(per // 2, (1 << 64) - 1, dtype=np.uint64),
                            rng.integers((1 << 64) - (1 << 44), (1 << 64) - 1, size=n, dtype=np.uint64)])
    keys = np.sort(v)
    q = queries_for(keys, 200000, 34, "random")
    want = oracle.lookup(keys, q, out_bytes=8)
    for g8 in ("0", "1"):
        monkeypatch.setenv("BS_BUCKET_G8", g8)
        idx = build(keys, variant=bs.KARY, out_bytes=8)
        check(bk_run(idx, q, 8), want, q, f"two-level {kind} g8={g8}")
        idx.close()


@pytest.mark.parametrize("kb", [4, 8])
def test_bucket_unaligned_buffers(kb):
    """Queries and results only key- / word-aligned (not 16-B aligned): the vector
    loads of the histogram pass and the vector stores of the unpartition pass
    fall back to scalar accesses."""
    keys = workload.gen_keys(3 * NB[kb] + 5, kb, seed=51)
    q = queries_for(keys, 5 * T + 3, 52, "random")
    want = oracle.lookup(keys, q, out_bytes=8)
    idx = build(keys, variant=bs.KARY, out_bytes=8)
    big = torch.zeros(q.size + 4, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
    dq = big[1:1 + q.size]                      # 4 / 8 B past a 16-B boundary
    dq.copy_(P.as_torch(q))
    obig = torch.full((q.size + 2,), -1, dtype=torch.int64, device="cuda")
    out = obig[1:1 + q.size]                    # 8 B past a 16-B boundary
    nb = bs.bs_workspace_bytes(idx, q.size, reorder=bs.REORDER_BUCKET)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    bs.bs_lookup_ws(idx, dq, q.size, out, None, ws, nb, reorder=bs.REORDER_BUCKET)
    torch.cuda.synchronize()
    check(P.to_numpy_unsigned(out, 8), want, q, f"unaligned kb={kb}")
    idx.close()
