"""The seeded generator (workload/): determinism, the P:61 recipe, golden checksums."""
import hashlib
import json
import os

import numpy as np
import pytest

import workload


def test_splitmix64_reference_values():
    # splitmix64 with state 0: first outputs of the canonical generator
    # (Steele, Lea, Flood 2014; Vigna's reference implementation), which adds
    # the golden gamma before mixing: next() = mix(state += gamma).
    v = workload.splitmix64(np.array([0, 0x9E3779B97F4A7C15], dtype=np.uint64))
    assert int(v[0]) == 0xE220A8397B1DCDAF
    assert int(v[1]) == 0x6E789E6AA1B965F4
    assert workload.splitmix64_int(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("kb,n", [(4, 1), (4, 1000), (4, 1 << 20), (8, 1 << 16), (8, 12345)])
def test_keys_unique_sorted(kb, n):
    k = workload.gen_keys(n, kb, seed=42)
    assert k.size == n and k.dtype == workload.key_dtype(kb)
    assert np.all(k[1:] > k[:-1])
    assert np.array_equal(k, workload.gen_keys(n, kb, seed=42))
    assert not np.array_equal(k, workload.gen_keys(n, kb, seed=43)) or n == 1


def test_keys_dense_domain_u32():
    # a quarter of a 2^16 domain is not available for u32, but a dense draw must
    # still be unique: n close to 2^32 is impractical, so test the subset path
    k = workload.gen_keys(1 << 22, 4, seed=1)
    assert np.all(k[1:] > k[:-1]) and k.size == 1 << 22
    # uniformity: top-byte histogram roughly flat
    h = np.bincount((k >> np.uint32(24)).astype(np.int64), minlength=256)
    assert h.min() > 0.8 * h.mean() and h.max() < 1.2 * h.mean()


def test_u64_keys_use_top_half():
    k = workload.gen_keys(1 << 16, 8, seed=2)
    assert (k >= np.uint64(1 << 63)).mean() > 0.4


def test_queries_hits_and_order():
    keys = workload.gen_keys(1000, 8, seed=5)
    q = workload.gen_queries(keys, 50000, seed=6, hit_ratio=1.0)
    assert np.isin(q, keys).all()
    qs = workload.gen_queries(keys, 50000, seed=6, hit_ratio=1.0, order="sorted")
    assert np.array_equal(np.sort(q), qs)
    q5 = workload.gen_queries(keys, 50000, seed=6, hit_ratio=0.5)
    frac = np.isin(q5, keys).mean()
    assert 0.47 < frac < 0.53
    q0 = workload.gen_queries(keys, 50000, seed=6, hit_ratio=0.0)
    assert np.isin(q0, keys).mean() < 0.001


def test_queries_slices_are_consistent():
    """Counter-based: shard j of the stream == the same slice of the whole stream."""
    keys = workload.gen_keys(1 << 12, 4, seed=9)
    whole = workload.gen_queries(keys, 40000, seed=10, hit_ratio=0.5)
    a = workload.gen_queries(keys, 15000, seed=10, hit_ratio=0.5, start=0)
    b = workload.gen_queries(keys, 25000, seed=10, hit_ratio=0.5, start=15000)
    assert np.array_equal(np.concatenate([a, b]), whole)


def test_golden_checksums(golden_dir):
    """Regression pin of the generator (written by tests/golden/make_golden.py)."""
    g = json.load(open(os.path.join(golden_dir, "workload_checksums.json")))
    for case in g["cases"]:
        keys = workload.gen_keys(case["n"], case["key_bytes"], seed=case["key_seed"])
        q = workload.gen_queries(keys, case["m"], seed=case["query_seed"], hit_ratio=case["hit_ratio"])
        assert hashlib.sha256(keys.tobytes()).hexdigest() == case["keys_sha256"]
        assert hashlib.sha256(q.tobytes()).hexdigest() == case["queries_sha256"]


# ---- workload/device.py: the same generator in torch int64 ops (CPU here, CUDA in test_gpu_workload.py)

def _bits(t):
    import torch
    return t.numpy().view(np.uint64 if t.dtype == torch.int64 else np.uint32)


@pytest.mark.parametrize("kb,n,seed", [(4, 1, 3), (4, 1000, 42), (4, 1 << 20, 7), (8, 1 << 16, 42),
                                       (8, 12345, 9), (4, 3 << 20, 11)])
def test_device_generator_keys_match_numpy(kb, n, seed):
    from workload import device as wd
    want = workload.gen_keys(n, kb, seed=seed)
    got = _bits(wd.gen_keys(n, kb, seed=seed, device="cpu"))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kb,n,m,hr,order,start", [
    (8, 1 << 12, 50000, 1.0, "random", 0), (8, 12345, 40000, 0.5, "random", 777),
    (4, 1000, 65536, 0.5, "random", 0), (4, 1 << 14, 30000, 1.0, "sorted", 5),
    (8, 3000, 20000, 0.0, "sorted", 0), (4, 7, 5000, 0.25, "random", 1 << 40)])
def test_device_generator_queries_match_numpy(kb, n, m, hr, order, start):
    import torch
    from workload import device as wd
    keys = workload.gen_keys(n, kb, seed=21)
    want = workload.gen_queries(keys, m, seed=22, hit_ratio=hr, order=order, start=start)
    tk = torch.from_numpy(keys.view(np.int64 if kb == 8 else np.int32))
    got = _bits(wd.gen_queries(tk, m, seed=22, hit_ratio=hr, order=order, start=start, chunk=1 << 13))
    assert np.array_equal(got, want)


def test_device_generator_unsigned_helpers():
    import torch
    from workload import device as wd
    x = np.array([0, 1, (1 << 63) - 1, 1 << 63, (1 << 64) - 1, 0x8000000000000001, 12345678901234567890],
                 dtype=np.uint64)
    t = torch.from_numpy(x.view(np.int64))
    assert np.array_equal(_bits(wd.sort_unsigned(t)), np.sort(x))
    for k in (1, 17, 31, 32, 63):
        assert np.array_equal(_bits(wd._lsr(t, k)), x >> np.uint64(k))
    for nn in (3, 1000, (1 << 33) + 7, 5):
        assert np.array_equal(wd._umod(t, nn).numpy().astype(np.uint64), x % np.uint64(nn))
    assert np.array_equal(_bits(wd.splitmix64(t)), workload.splitmix64(x))


def test_device_generator_range_keys():
    """Config-5 shard keys: unique, ascending, inside [lo, hi), roughly uniform."""
    from workload import device as wd
    N = 8
    for s in (0, 3, 7):
        lo, hi = s << 61, (s + 1) << 61
        k = _bits(wd.gen_keys_range(1 << 16, lo, hi, seed=5, shard=s, device="cpu"))
        assert k.size == 1 << 16 and np.all(k[1:] > k[:-1])
        assert int(k[0]) >= lo and int(k[-1]) < hi
        h = np.bincount(((k - np.uint64(lo)) >> np.uint64(61 - 4)).astype(np.int64), minlength=16)
        assert h.min() > 0.8 * h.mean() and h.max() < 1.2 * h.mean()
    assert N == 8
