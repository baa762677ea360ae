"""K-ary schedule (kary_mode) vs build size, one B200: 2^27 random hit
queries, median-of-3 CUDA-event time, sampled parity, the index default
layout otherwise.

python tools/mode_sweep.py --kb 8 --lo 16 --hi 26 --modes 2,3,6,7 > gpurun_out/modes.jsonl
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
import workload  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402
from tools.size_sweep import time_launch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kb", type=int, default=8)
    ap.add_argument("--lo", type=int, default=16)
    ap.add_argument("--hi", type=int, default=26)
    ap.add_argument("--step", type=int, default=2)
    ap.add_argument("--modes", default="2,3,6,7")
    ap.add_argument("--kc", default="5/16", help="K/C pairs, e.g. 5/16,5/8,5/4")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    kb, m = a.kb, 1 << 27
    out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
    for lg in range(a.lo, a.hi + 1, a.step):
        n = 1 << lg
        keys = workload.gen_keys(n, kb)
        q = workload.gen_queries(keys, m)
        dk, dq = P.as_torch(keys), P.as_torch(q)
        samp = np.random.default_rng(lg).integers(0, m, size=1 << 12)
        want = oracle.lookup(keys, q[samp], out_bytes=kb)
        for kc in a.kc.split(","):
            K, C = (int(x) for x in kc.split("/"))
            idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, k=K, leaf_chunk=C))
            for mode in (int(x) for x in a.modes.split(",")):
                ms = time_launch(lambda: bs.bs_lookup_ex(idx, dq, m, out, None, kary_mode=mode), 2, 3)
                ok = bool(np.array_equal(P.to_numpy_unsigned(out, kb)[samp], want))
                print(json.dumps({"log2n": lg, "key_bytes": kb, "K": K, "C": C, "kary_mode": mode, "ms": ms,
                                  "G_lookups_per_s": m / ms / 1e6, "ok": ok}), flush=True)
            idx.close()
        del dk, dq
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
