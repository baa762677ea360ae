"""bs_merge (batch inserts, include/bs.h): the merged index's
sorted array is bit-exactly np.sort(a ++ delta) and every variant's lookups on
it equal the oracle over that array — duplicates, keys below/above the old
range, the MAX key, an empty and a full-size delta, sorted and unsorted."""
import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def _delta(keys, m, seed):
    rng = np.random.default_rng(seed)
    dt = keys.dtype
    info = np.iinfo(dt)
    ext = np.array([0, info.max, keys[0], keys[-1]], dtype=dt)                      # extremes
    dup = keys[rng.integers(0, keys.size, size=m // 3)]                             # duplicates of old keys
    rnd = rng.integers(0, info.max, size=max(m - dup.size - ext.size, 0), dtype=dt, endpoint=True)
    d = np.concatenate([ext, dup, rnd])[:m]
    rng.shuffle(d)
    return d.astype(dt)


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("variant", [bs.NAIVE, bs.OPT, bs.KARY])
@pytest.mark.parametrize("m", [0, 1, 4097, 150001])
def test_merge_parity(kb, variant, m):
    keys = workload.gen_keys(100003, kb, seed=51)
    idx = bs.bs_build(P.as_torch(keys), keys.size, bs.bs_layout_default(key_bytes=kb, out_bytes=8, variant=variant))
    delta = _delta(keys, m, seed=52 + m)
    merged_np = np.sort(np.concatenate([keys, delta]))
    assert delta.size == m
    new = bs.bs_merge(idx, P.as_torch(delta) if m else None, m)
    assert new.info["n"] == merged_np.size
    assert np.array_equal(bs.bs_export(new, bs.EXPORT_SORTED), merged_np)
    q = np.concatenate([workload.gen_queries(merged_np, 60000, seed=53, hit_ratio=0.7), delta[:1000]])
    out = torch.empty(q.size, dtype=torch.int64, device="cuda")
    bs.bs_lookup(new, P.as_torch(q), q.size, out)
    torch.cuda.synchronize()
    assert np.array_equal(P.to_numpy_unsigned(out, 8), oracle.lookup(merged_np, q, out_bytes=8))
    # the old index is untouched
    bs.bs_lookup(idx, P.as_torch(q), q.size, out)
    torch.cuda.synchronize()
    assert np.array_equal(P.to_numpy_unsigned(out, 8), oracle.lookup(keys, q, out_bytes=8))
    new.close()
    idx.close()


@pytest.mark.parametrize("variant", [bs.OPT, bs.KARY])
def test_merge_u32_out4(variant):
    keys = workload.gen_keys(30011, 4, seed=71)
    idx = bs.bs_build(P.as_torch(keys), keys.size, bs.bs_layout_default(key_bytes=4, out_bytes=4, variant=variant))
    delta = _delta(keys, 9001, seed=72)
    new = bs.bs_merge(idx, P.as_torch(delta), delta.size)
    merged_np = np.sort(np.concatenate([keys, delta]))
    q = np.concatenate([workload.gen_queries(merged_np, 40000, seed=73, hit_ratio=0.5), delta])
    out = torch.empty(q.size, dtype=torch.int32, device="cuda")
    bs.bs_lookup(new, P.as_torch(q), q.size, out)
    torch.cuda.synchronize()
    assert np.array_equal(P.to_numpy_unsigned(out, 4), oracle.lookup(merged_np, q, out_bytes=4))
    new.close()
    idx.close()


def test_merge_sorted_delta_flag():
    keys = workload.gen_keys(5000, 8, seed=61)
    idx = bs.bs_build(P.as_torch(keys), keys.size, bs.bs_layout_default(key_bytes=8, out_bytes=8))
    delta = _delta(keys, 3000, seed=62)
    ds = np.sort(delta)
    new = bs.bs_merge(idx, P.as_torch(ds), ds.size, delta_sorted=True)
    assert np.array_equal(bs.bs_export(new, bs.EXPORT_SORTED), np.sort(np.concatenate([keys, delta])))
    new.close()
    with pytest.raises(bs.BsError) as e:   # claimed sorted but is not
        bs.bs_merge(idx, P.as_torch(delta), delta.size, delta_sorted=True)
    assert e.value.code == -6
    idx.close()
