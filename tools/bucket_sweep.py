"""Lookup throughput vs build size, random batch: the K-ary kernel (random order,
the round-1 default) vs BS_REORDER_BUCKET (the key-range partition, DESIGN.md
§6.11) — the paper's Fig. 11 analogue for the two modes on one B200.

python tools/bucket_sweep.py --kb 8 --lo 20 --hi 30 > gpurun_out/bucket_sweep.jsonl
For each n = 2^lo .. 2^hi (step 2): m = 2^27 uniform random hit queries (the
workload generator on the device); median of 5 timed launches after 2 warm-ups
(CUDA events); each mode checked on a 2^12 sample against the oracle.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
import workload.device as wd  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def time_launch(fn, warmup, reps):
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kb", type=int, default=8)
    ap.add_argument("--lo", type=int, default=20)
    ap.add_argument("--hi", type=int, default=30)
    ap.add_argument("--step", type=int, default=2)
    ap.add_argument("--m-log2", type=int, default=27)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    kb, m = a.kb, 1 << a.m_log2
    for lg in range(a.lo, a.hi + 1, a.step):
        n = 1 << lg
        dk = wd.gen_keys(n, kb, device="cuda")
        dq = wd.gen_queries(dk, m)
        out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
        keys = P.to_numpy_unsigned(dk, kb)
        samp = np.random.default_rng(lg).integers(0, m, size=1 << 12)
        qs = P.to_numpy_unsigned(dq[torch.from_numpy(samp).cuda()], kb)
        want = oracle.lookup(keys, qs, out_bytes=kb)
        idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb))
        nb = bs.bs_workspace_bytes(idx, m, reorder=bs.REORDER_BUCKET)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        modes = [("kary", lambda: bs.bs_lookup_ex(idx, dq, m, out, None, reorder=bs.REORDER_NONE)),
                 ("bucket", lambda: bs.bs_lookup_ws(idx, dq, m, out, None, ws, nb, reorder=bs.REORDER_BUCKET))]
        for name, fn in modes:
            ms = time_launch(fn, 2, 5)
            ok = bool(np.array_equal(P.to_numpy_unsigned(out, kb)[samp], want))
            print(json.dumps({"n": n, "log2n": lg, "key_bytes": kb, "m": m, "mode": name, "ms": ms,
                              "G_lookups_per_s": m / ms / 1e6, "ok": ok}), flush=True)
        idx.close()
        del dk, dq, out, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
