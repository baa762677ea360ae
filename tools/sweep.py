"""Launch-knob sweeps on one GPU (Fig. 4 / 6 / 8 / 10 analogues on B200).

python tools/sweep.py --config config3 --what kary,opt,naive [--order random] > gpurun_out/sweep.jsonl
Each line: one (variant, knobs) point, ms per 2^27-lookup batch (CUDA events,
median of --reps after --warmup) and lookups/s; a sampled oracle check per
point.  Not the bench contract — bench.py is.
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def time_launch(fn, warmup, reps):
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--order", default="random")
    ap.add_argument("--what", default="kary,opt,naive")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--kc", default="")
    ap.add_argument("--hints", default="3")
    ap.add_argument("--modes", default="1,0")
    ap.add_argument("--tr", default="", help="threads/R pairs for kary, e.g. 512/8,1024/4")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    keys, q, desc = bench.make_inputs(args.config, args.order, 0)
    n, kb, m = bench.CONFIGS[args.config][:3]
    dk, dq = P.as_torch(keys), P.as_torch(q)
    out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
    samp = np.random.default_rng(7).integers(0, m, size=1 << 12)
    want = oracle.lookup(keys, q[samp])

    def emit(rec, ms, ok):
        rec.update(ms=ms, glookups_per_s=m / ms / 1e6, ok=ok, config=args.config, order=args.order)
        print(json.dumps(rec), flush=True)

    def measure(idx, rec, **launch):
        def fn():
            bs.bs_lookup_ex(idx, dq, m, out, None, **launch)
        try:
            ms = time_launch(fn, args.warmup, args.reps)
        except bs.BsError as e:
            rec.update(error=str(e))
            print(json.dumps(rec), flush=True)
            return
        got = P.to_numpy_unsigned(out, kb)[samp]
        emit(rec, ms, bool(np.array_equal(got, want)))

    what = args.what.split(",")
    if "naive" in what:
        idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, variant=bs.NAIVE))
        for t in (64, 128, 256, 512, 1024):
            measure(idx, {"variant": "naive", "threads": t}, variant=bs.NAIVE, threads=t)
        idx.close()
    if "kary" in what:
        kcs = [(17, 16), (9, 8), (5, 4), (17, 8), (9, 16), (33, 32), (5, 8), (17, 32)]
        if args.kc:
            kcs = [tuple(map(int, x.split("/"))) for x in args.kc.split(",")]
        for K, C in kcs:
            idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, variant=bs.KARY, k=K, leaf_chunk=C))
            info = idx.info
            grid = itertools.product([256, 512, 1024], [1, 2, 4, 8], [bs.STATIC, bs.DYNAMIC], [1, 0], [3, 0])
            if args.quick:
                hl = [int(h) for h in args.hints.split(",")]
                trs = [tuple(map(int, x.split("/"))) for x in args.tr.split(",")] if args.tr else \
                    [(512, 4), (512, 8), (1024, 4), (256, 8)]
                grid = [(t, R, bs.STATIC, 1, h) for (t, R) in trs for h in hl]
            modes = [int(x) for x in args.modes.split(",")]
            for mode in modes:
                for t, R, sched, pin, hints in grid:
                    if sched == bs.DYNAMIC and pin:
                        continue
                    rec = {"variant": "kary", "mode": mode, "K": K, "C": C, "threads": t, "R": R, "sched": sched,
                           "pin": pin, "hints": hints, "levels": info["kary_levels"]}
                    measure(idx, rec, variant=bs.KARY, threads=t, nreg=R, schedule=sched, use_pinned=pin,
                            cache_hints=hints, kary_mode=mode)
            idx.close()
    if "ladder" in what:
        # the paper's §4 optimisation ladder (Figs. 4/6/8 analogues): scheduling,
        # steps- vs full-pinning, lookup- vs full-reordering, on the OPT kernel
        idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, variant=bs.OPT))
        measure(idx, {"variant": "naive", "step": "naive dynamic 256"}, variant=bs.NAIVE, threads=256)
        for t, nreg in ((256, 4), (256, 8), (512, 4), (1024, 2)):
            steps = [("static", dict(use_pinned=0, reorder=0, pin_partial=0)),
                     ("static+steps-pinning", dict(use_pinned=1, reorder=0, pin_partial=0)),
                     ("static+full-pinning", dict(use_pinned=1, reorder=0, pin_partial=1)),
                     ("+lookup-reordering", dict(use_pinned=1, reorder=1, pin_partial=1)),
                     ("+full-reordering", dict(use_pinned=1, reorder=2, pin_partial=1))]
            for name, kw in steps:
                rec = {"variant": "opt", "step": name, "threads": t, "nreg": nreg}
                measure(idx, rec, variant=bs.OPT, threads=t, nreg=nreg, schedule=bs.STATIC, **kw)
        idx.close()
    if "opt" in what:
        idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, variant=bs.OPT))
        grid = itertools.product([128, 256, 512, 1024], [1, 2, 4, 8, 16], [0, 1, 2], [1, 0], [bs.STATIC])
        if args.quick:
            grid = itertools.product([256, 512], [4, 8], [0, 2], [1], [bs.STATIC])
        for t, nreg, reorder, pin, sched in grid:
            rec = {"variant": "opt", "threads": t, "nreg": nreg, "reorder": reorder, "pin": pin, "sched": sched}
            measure(idx, rec, variant=bs.OPT, threads=t, nreg=nreg, reorder=reorder, use_pinned=pin,
                    pin_partial=1, schedule=sched)
        idx.close()


if __name__ == "__main__":
    main()
