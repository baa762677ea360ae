"""Pins for the CPU oracle (oracle/oracle.c) — independent of the oracle itself.

Each pin is chosen so that a plausible mistake fails at least one of them:
  * brute-force rank count  #{i : a[i] < q}  (dropped/extra term, off-by-one,
    '<=' instead of '<' -> upper bound, wrong hit test);
  * numpy.searchsorted(side='left') on uint64 incl. keys >= 2^63 (signed
    compare mistakes);
  * the invariant a[lb-1] < q <= a[lb], which determines lb uniquely;
  * the paper's / SPEC's worked examples (tests/golden/);
  * the miss-bit position per output width (transposed encodings).
"""
import ctypes
import json
import os

import numpy as np
import pytest

import oracle
import workload


def brute(keys, queries, out_bytes):
    """Brute force on tiny inputs: lb = number of keys < q; hit iff a[lb] == q."""
    k = keys.astype(np.uint64)
    q = queries.astype(np.uint64)
    lb = (k[None, :] < q[:, None]).sum(axis=1).astype(np.uint64)
    hit = np.zeros(q.size, dtype=bool)
    inb = lb < k.size
    hit[inb] = k[lb[inb].astype(np.int64)] == q[inb]
    mb = np.uint64(1 << (8 * out_bytes - 1))
    out = np.where(hit, lb, lb | mb)
    return out.astype({4: np.uint32, 8: np.uint64}[out_bytes])


def random_sorted(rng, n, dtype, dup_prob):
    info = np.iinfo(dtype)
    mode = rng.integers(0, 3)
    if mode == 0:      # full domain
        v = rng.integers(0, int(info.max), size=n, dtype=np.uint64, endpoint=True).astype(dtype)
    elif mode == 1:    # narrow range -> many duplicates and gaps
        v = rng.integers(0, 4 * n + 3, size=n, dtype=np.uint64).astype(dtype)
    else:              # top of the domain (>= 2^63 for u64) incl. MAX
        v = (info.max - rng.integers(0, 3 * n + 1, size=n, dtype=np.uint64)).astype(dtype)
    if dup_prob > 0 and n > 1:
        d = rng.random(n) < dup_prob
        src = rng.integers(0, n, size=n)
        v = np.where(d, v[src], v)
    return np.sort(v)


def queries_for(rng, keys, extra=100):
    dt = keys.dtype
    mx = np.iinfo(dt).max
    parts = [keys,
             np.array([0, 1, mx, mx - 1], dtype=dt),
             rng.integers(0, int(mx), size=extra, dtype=np.uint64, endpoint=True).astype(dt)]
    lo = keys[keys > 0] - dt.type(1)
    hi = keys[keys < mx] + dt.type(1)
    parts += [lo[: extra], hi[: extra]]
    if keys.size:
        parts.append(np.array([keys[0], keys[-1]], dtype=dt))
    q = np.concatenate(parts).astype(dt)
    rng.shuffle(q)
    return q


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64])
def test_oracle_vs_brute_force(dtype):
    """>= 1000 random sorted arrays, n in [1, 2^12], duplicates, all present keys
    plus >= 100 absent ones (below-min, above-max, gaps, 0, MAX)."""
    rng = np.random.default_rng(1234 + np.dtype(dtype).itemsize)
    for trial in range(520):
        n = int(np.exp(rng.uniform(0, np.log(4096))))
        n = max(1, min(n, 4096))
        keys = random_sorted(rng, n, dtype, dup_prob=[0.0, 0.3][trial % 2])
        q = queries_for(rng, keys)
        for ob in (8, 4):
            got = oracle.lookup(keys, q, out_bytes=ob)
            exp = brute(keys, q, ob)
            assert np.array_equal(got, exp), (trial, n, ob)


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64])
def test_oracle_vs_searchsorted(dtype):
    """Library special case (numpy.searchsorted side='left', unsigned dtypes)."""
    rng = np.random.default_rng(99)
    for n in (1, 2, 3, 7, 8, 9, 1000, 1 << 14, (1 << 14) + 3):
        keys = random_sorted(rng, n, dtype, dup_prob=0.2)
        q = queries_for(rng, keys, extra=1000)
        lb = np.searchsorted(keys, q, side="left").astype(np.uint64)
        got = oracle.lookup(keys, q, out_bytes=8)
        assert np.array_equal(got & np.uint64((1 << 63) - 1), lb)


def test_oracle_invariant_on_generated_workloads():
    """a[lb-1] < q <= a[lb] (a[-1] = -inf, a[n] = +inf) fixes lb uniquely."""
    for kb, n, m, hr in ((4, 1 << 10, 1 << 16, 0.5), (8, 1 << 16, 1 << 18, 0.5), (8, 12345, 1 << 17, 1.0)):
        keys = workload.gen_keys(n, kb, seed=7)
        q = workload.gen_queries(keys, m, seed=8, hit_ratio=hr)
        out = oracle.lookup(keys, q)
        mb = np.uint64(oracle.miss_bit(kb))
        o = out.astype(np.uint64)
        lb = (o & ~mb).astype(np.int64)
        hit = (o & mb) == 0
        assert lb.min() >= 0 and lb.max() <= n
        k64 = keys.astype(np.uint64)
        q64 = q.astype(np.uint64)
        left_ok = (lb == 0) | (k64[np.maximum(lb - 1, 0)] < q64)
        right_ok = (lb == n) | (q64 <= k64[np.minimum(lb, n - 1)])
        assert left_ok.all() and right_ok.all()
        at = k64[np.minimum(lb, n - 1)]
        assert np.array_equal(hit, (lb < n) & (at == q64))
        if hr == 1.0:
            assert hit.all()


def test_spec_primes_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_primes.json")))
    for dt in (np.uint32, np.uint64):
        keys = np.array(g["keys"], dtype=dt)
        for c in g["cases"]:
            assert oracle.lower_bound(keys, c["q"]) == c["lb"]
            out = int(oracle.lookup(keys, np.array([c["q"]], dtype=dt))[0])
            mb = oracle.miss_bit(keys.dtype.itemsize)
            assert (out & (mb - 1)) == c["lb"]
            assert ((out & mb) == 0) == c["hit"]
        d = g["duplicates"]
        out = int(oracle.lookup(np.array(d["keys"], dtype=dt), np.array([d["q"]], dtype=dt))[0])
        assert out == d["lb"]


def test_fig5_identity_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "fig3_fig5_n14.json")))
    keys = np.array(g["keys"], dtype=np.uint32)
    assert oracle.lower_bound(keys, g["query"]) == g["offset"]


def test_miss_bit_width_and_values():
    keys = np.array([10, 20, 30], dtype=np.uint64)
    q = np.array([5, 10, 15, 30, 31], dtype=np.uint64)
    o8 = oracle.lookup(keys, q, out_bytes=8)
    assert list(o8) == [0 | (1 << 63), 0, 1 | (1 << 63), 2, 3 | (1 << 63)]
    o4 = oracle.lookup(keys, q, out_bytes=4)
    assert list(o4) == [0 | (1 << 31), 0, 1 | (1 << 31), 2, 3 | (1 << 31)]
    k32 = keys.astype(np.uint32)
    assert list(oracle.lookup(k32, q.astype(np.uint32), out_bytes=8)) == list(o8)


def test_oracle_argument_errors():
    lib = oracle._load()
    k = np.zeros(4, dtype=np.uint64)
    q = np.zeros(1, dtype=np.uint64)
    out = np.zeros(1, dtype=np.uint64)
    # n == 0 rejected; u32 output with n >= 2^31 rejected before any access
    assert lib.oracle_lookup(k.ctypes.data, 0, 8, q.ctypes.data, 1, out.ctypes.data, 8) == -1
    assert lib.oracle_lookup(k.ctypes.data, 1 << 31, 8, q.ctypes.data, 1, out.ctypes.data, 4) == -1
    assert lib.oracle_lookup(k.ctypes.data, 4, 5, q.ctypes.data, 1, out.ctypes.data, 8) == -1


def test_oracle_mt_matches_single():
    keys = workload.gen_keys(1 << 15, 8, seed=3)
    q = workload.gen_queries(keys, 100003, seed=4, hit_ratio=0.7)
    a = oracle.lookup(keys, q, threads=1)
    for t in (2, 3, 8, 200000):
        assert np.array_equal(oracle.lookup(keys, q, threads=t), a)


def test_mutation_sensitivity_of_pins():
    """A wrong lower bound (upper bound, '<=' for '<') must fail the brute-force pin."""
    keys = np.array([1, 3, 3, 3, 7], dtype=np.uint64)
    q = np.array([3], dtype=np.uint64)
    upper = np.searchsorted(keys, q, side="right")
    assert int(brute(keys, q, 8)[0]) == 1 != int(upper[0])
    assert int(oracle.lookup(keys, q)[0]) == 1
