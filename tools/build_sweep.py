"""Build time per stage vs n (Figs. 12-13):
bs_build of the default K-ary index over n u64 (and u32) keys, sorted input
(sortedness check) and unsorted input (the library's radix sort), median of
--reps builds after a warm-up build.  Stage times are device times from event
pairs around each group of build kernels (bs_info.build_stage_us), so
allocation is excluded; wall = host time of the synchronous call.  One JSON
line per (key width, n, input order).

python tools/build_sweep.py [--lo 15] [--hi 30] [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workload  # noqa: E402
from workload import device as wd  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402

STAGES = ["sort", "check", "pinned_table", "separators", "images"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lo", type=int, default=15)
    ap.add_argument("--hi", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kb", type=int, nargs="*", default=[8, 4])
    a = ap.parse_args()
    for kb in a.kb:
        for lg in range(a.lo, (a.hi if kb == 8 else min(a.hi, 29)) + 1):
            n = 1 << lg
            keys = wd.gen_keys(n, kb, seed=workload.KEY_SEED, device="cuda")
            g = torch.Generator(device="cuda")
            g.manual_seed(lg)
            shuffled = keys[torch.randperm(n, device="cuda", generator=g)]
            for order, src, sorted_flag in (("sorted", keys, 1), ("unsorted", shuffled, 0)):
                lay = bs.bs_layout_default(key_bytes=kb, out_bytes=kb, input_sorted=sorted_flag)
                bs.bs_build(src, n, lay).close()          # warm-up
                rows = []
                for _ in range(a.reps):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    idx = bs.bs_build(src, n, lay)
                    wall = (time.perf_counter() - t0) * 1e3
                    info = idx.info
                    rows.append((wall, info))
                    idx.close()
                med = lambda xs: statistics.median(xs)  # noqa: E731
                st = {s: med([r[1]["build_stage_us"][i] for r in rows]) / 1e3 for i, s in enumerate(STAGES)}
                info = rows[0][1]
                print(json.dumps({"key_bytes": kb, "log2n": lg, "n": n, "input": order,
                                  "stage_ms": st, "kernels_ms": sum(st.values()),
                                  "device_span_ms": med([r[1]["build_ms"] for r in rows]),
                                  "wall_ms": med([r[0] for r in rows]),
                                  "footprint_over_array": info["footprint_bytes"] / info["array_bytes"],
                                  "leaf_chunk": info["leaf_chunk"], "kary_levels": info["kary_levels"]}), flush=True)
            del keys, shuffled
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
