"""Lookup throughput vs build size (the paper's Fig. 1a / Fig. 11 analogue) and
build time / footprint (Figs. 12-13 analogue) on one B200.

python tools/size_sweep.py --kb 4 --lo 15 --hi 29 > gpurun_out/size_sweep.jsonl
For each n = 2^lo .. 2^hi (step 2): m = 2^27 uniform random hit queries; the
naive kernel (Listing 1), the OPT kernel (static + steps-pinning, 512 x 4) and
the K-ary bench kernel (mode 6) — each checked on a sample against the oracle.
Lines: {"n", "variant", "ms", "G_lookups_per_s", "build_ms_sorted_input",
"build_ms_unsorted_input", "footprint_bytes", "ok"}; build times are host wall
times of the synchronous bs_build (median of 3 after a warm-up build).
"""
from __future__ import annotations

import argparse
import json
import os
import time
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
import workload  # noqa: E402
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
    ap.add_argument("--kb", type=int, default=4)
    ap.add_argument("--lo", type=int, default=15)
    ap.add_argument("--hi", type=int, default=29)
    ap.add_argument("--step", type=int, default=2)
    ap.add_argument("--m-log2", type=int, default=27)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--c", type=int, default=0, help="leaf chunk; 0 = the layout's auto choice")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    kb, m = a.kb, 1 << a.m_log2
    out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
    for lg in range(a.lo, a.hi + 1, a.step):
        n = 1 << lg
        keys = workload.gen_keys(n, kb)
        q = workload.gen_queries(keys, m)
        dk, dq = P.as_torch(keys), P.as_torch(q)
        dk_perm = dk[torch.randperm(n, device="cuda")]
        samp = np.random.default_rng(lg).integers(0, m, size=1 << 12)
        want = oracle.lookup(keys, q[samp], out_bytes=kb)
        runs = [("naive", dict(variant=bs.NAIVE), dict(variant=bs.NAIVE, threads=256)),
                ("opt", dict(variant=bs.OPT), dict(variant=bs.OPT, threads=512, nreg=4, use_pinned=1, pin_partial=0,
                                                   reorder=0, schedule=bs.STATIC)),
                ("kary", dict(variant=bs.KARY, k=a.k, leaf_chunk=a.c), dict(variant=bs.KARY))]
        for name, lay_kw, launch_kw in runs:
            # build time (Fig. 13 analogue): host wall time of the synchronous
            # bs_build, median of 3 after one warm-up build; input already
            # sorted (copy + check + auxiliary levels) and unsorted (+ radix sort)
            bt = {}
            for srt in (1, 0):
                ts = []
                for r in range(4):
                    lay = bs.bs_layout_default(key_bytes=kb, out_bytes=kb, input_sorted=srt, **lay_kw)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    ib = bs.bs_build(dk if srt else dk_perm, n, lay)
                    ts.append((time.perf_counter() - t0) * 1e3)
                    ib.close()
                bt[srt] = float(np.median(ts[1:]))
            idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, **lay_kw))
            info = idx.info

            def fn():
                bs.bs_lookup_ex(idx, dq, m, out, None, **launch_kw)
            ms = time_launch(fn, 2, 3)
            ok = bool(np.array_equal(P.to_numpy_unsigned(out, kb)[samp], want))
            print(json.dumps({"n": n, "log2n": lg, "key_bytes": kb, "variant": name, "ms": ms,
                              "G_lookups_per_s": m / ms / 1e6, "build_ms_sorted_input": bt[1],
                              "build_ms_unsorted_input": bt[0],
                              "footprint_bytes": info["footprint_bytes"], "array_bytes": info["array_bytes"],
                              "leaf_chunk": info["leaf_chunk"], "kary_mode": bs.bs_launch_default(idx).kary_mode,
                              "ok": ok}), flush=True)
            idx.close()
        del dk, dq, dk_perm
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
