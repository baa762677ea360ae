"""u64 keys confined to a narrow range: every key < 2^32
(all high words equal) and < 2^40, 2^26 keys, 2^27 random hit queries, the
default lookup (bench.py's launch configuration) vs uniform u64 keys.  CUDA
events, median of --reps after warm-up; parity on a sample.  One JSON line per
distribution.

python tools/tie_bench.py [--reps 10] [--n-log2 26] [--m-log2 27]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workload  # noqa: E402
from workload import device as wd  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--n-log2", type=int, default=26)
    ap.add_argument("--m-log2", type=int, default=27)
    a = ap.parse_args()
    n, m = 1 << a.n_log2, 1 << a.m_log2
    s = torch.cuda.Stream()
    for name, hi in (("uniform u64", 1 << 64), ("u64 < 2^40", 1 << 40), ("u64 < 2^32", 1 << 32)):
        keys = wd.gen_keys_range(n, 0, hi, workload.KEY_SEED, 0, device="cuda")
        q = wd.gen_queries(keys, m, seed=workload.QUERY_SEED)
        out = torch.empty(m, dtype=torch.int64, device="cuda")
        idx = bs.bs_build(keys, n, bs.bs_layout_default())
        with torch.cuda.stream(s):
            for _ in range(3):
                bs.bs_lookup(idx, q, m, out, s)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            bs.bs_lookup(idx, q, m, out, s)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        kh = keys.cpu().numpy().view(np.uint64)
        samp = np.random.default_rng(1).integers(0, m, size=1 << 14)
        qh = q.cpu().numpy().view(np.uint64)[samp]
        ok = bool(np.array_equal(P.to_numpy_unsigned(out, 8)[samp], oracle.lookup(kh, qh, out_bytes=8)))
        ms = statistics.median(ts)
        print(json.dumps({"keys": name, "n": n, "m": m, "ms": ms, "G_lookups_per_s": m / ms / 1e6,
                          "parity_sample_ok": ok, "kary_mode": bs.bs_launch_default(idx).kary_mode}), flush=True)
        idx.close()
        del keys, q, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
