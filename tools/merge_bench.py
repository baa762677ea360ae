"""Cost of batch inserts and deletes (P:254 outlook): bs_merge of a random
delta into the config-3 index (2^26 u64 keys, K-ary layout) vs rebuilding
from the unsorted concatenation (bs_build, library radix sort).  Host wall
time of the synchronous calls, median of 3 after a warm-up.  One JSON line per
delta size; the merged array is checked against np.sort on a sample.

python tools/merge_bench.py > gpurun_out/merge.jsonl
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_01576_b200 as P  # noqa: E402
import workload  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def wall(fn, reps=3):
    fn().close()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ix = fn()
        ts.append((time.perf_counter() - t0) * 1e3)
        ix.close()
    return statistics.median(ts)


def main():
    torch.cuda.set_device(0)
    n = 1 << 26
    keys = workload.gen_keys(n, 8, seed=workload.KEY_SEED)
    dk = P.as_torch(keys)
    lay = bs.bs_layout_default(key_bytes=8, out_bytes=8)
    idx = bs.bs_build(dk, n, lay)
    rng = np.random.default_rng(7)
    for frac in (0.001, 0.01, 0.1, 1.0):
        m = int(n * frac)
        delta = rng.integers(0, np.iinfo(np.uint64).max, size=m, dtype=np.uint64, endpoint=True)
        dd = P.as_torch(delta)
        t_merge = wall(lambda: bs.bs_merge(idx, dd, m))
        cat = torch.cat([dk, dd])
        lay_u = bs.bs_layout_default(key_bytes=8, out_bytes=8, input_sorted=0)
        t_rebuild = wall(lambda: bs.bs_build(cat, n + m, lay_u))
        new = bs.bs_merge(idx, dd, m)
        got = bs.bs_export(new, bs.EXPORT_SORTED)
        want = np.sort(np.concatenate([keys, delta]))
        ok = bool(np.array_equal(got, want))
        new.close()
        print(json.dumps({"n": n, "m": m, "merge_ms": t_merge, "rebuild_from_unsorted_ms": t_rebuild,
                          "speedup": t_rebuild / t_merge, "merged_array_exact": ok}), flush=True)
        del cat, dd
        torch.cuda.empty_cache()
    # batch deletes: erase a random subset of the keys (plus as many absent values)
    for frac in (0.001, 0.01, 0.1):
        m = int(n * frac)
        dele = np.concatenate([keys[rng.integers(0, n, size=m // 2)],
                               rng.integers(0, np.iinfo(np.uint64).max, size=m - m // 2, dtype=np.uint64,
                                            endpoint=True)])
        dd = P.as_torch(dele)
        t_erase = wall(lambda: bs.bs_erase(idx, dd, m))
        new = bs.bs_erase(idx, dd, m)
        got = bs.bs_export(new, bs.EXPORT_SORTED)
        ok = bool(np.array_equal(got, keys[~np.isin(keys, dele)]))
        new.close()
        print(json.dumps({"n": n, "m_delete": m, "erase_ms": t_erase, "erased_array_exact": ok}), flush=True)
    idx.close()


if __name__ == "__main__":
    main()
