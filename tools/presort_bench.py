"""SURVEY §8f f3 comparator: does a GLOBAL pre-sort of the batch pay for itself?
(the paper's local reordering is a cheap approximation of sorting
all lookups, which it calls too expensive; Fig. 1b shows pre-sorted lookups
are much faster.)  Config 3 (2^26 u64 keys, 2^27 random queries), one B200:

  random      bs_lookup on the random batch (the bench step)
  presorted   bs_lookup on an already sorted batch (sort not timed; Fig. 1b)
  sort+lookup+unsort
              device radix sort of (key, index) pairs (torch.sort -> CUB, a
              library sort: a comparator, not a product path), bs_lookup on
              the sorted keys, scatter of the results back to query order

CUDA events on one stream, median of --reps.  One JSON line per row; the
sort+lookup+unsort row is checked on a sample against the oracle.
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
import paper_2506_01576_b200 as P  # noqa: E402
import workload  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402

SIGN = -(1 << 63)


def timed(fn, reps):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n, m = 1 << 26, 1 << 27
    keys = workload.gen_keys(n, 8, seed=workload.KEY_SEED)
    q = workload.gen_queries(keys, m, seed=workload.QUERY_SEED)
    qs = np.sort(q)
    dk, dq, dqs = P.as_torch(keys), P.as_torch(q), P.as_torch(qs)
    idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=8, out_bytes=8))
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    res_sorted = torch.empty_like(out)
    sign = torch.tensor(SIGN, dtype=torch.int64, device="cuda")
    rows = [("random", timed(lambda: bs.bs_lookup(idx, dq, m, out), a.reps)),
            ("presorted (sort not timed)", timed(lambda: bs.bs_lookup(idx, dqs, m, out), a.reps))]

    def sort_lookup_unsort():
        # unsigned order = signed order of (bits ^ 2^63)
        sv, perm = torch.sort(dq ^ sign)
        sk = sv ^ sign
        bs.bs_lookup(idx, sk, m, res_sorted)
        out.scatter_(0, perm, res_sorted)

    t_sort = timed(lambda: torch.sort(dq ^ sign), a.reps)
    rows.append(("sort only (torch.sort of 2^27 int64 + indices)", t_sort))
    rows.append(("sort+lookup+unsort", timed(sort_lookup_unsort, a.reps)))
    sort_lookup_unsort()
    torch.cuda.synchronize()
    samp = np.random.default_rng(5).integers(0, m, size=1 << 14)
    ok = bool(np.array_equal(P.to_numpy_unsigned(out, 8)[samp], oracle.lookup(keys, q[samp], out_bytes=8)))
    for name, ms in rows:
        print(json.dumps({"row": name, "ms": ms, "G_lookups_per_s": m / ms / 1e6, "n": n, "m": m,
                          "parity_sample_ok": ok}), flush=True)
    idx.close()


if __name__ == "__main__":
    main()
