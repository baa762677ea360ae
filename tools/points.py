"""Launch a list of K-ary configurations twice each (for ncu metric collection).

python tools/points.py --pts 5/8/2/1024/2,9/8/2/1024/4 [--config config3]
Each point K/C/mode/threads/I[/hints]: build (once per K/C), then 2 launches;
ncu -k regex:k_kary collects both (use the second).  Prints the launch order.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config3")
ap.add_argument("--order", default="random")
ap.add_argument("--pts", required=True)
a = ap.parse_args()
torch.cuda.set_device(0)
keys, q, _ = bench.make_inputs(a.config, a.order, 0)
n, kb, m = bench.CONFIGS[a.config][:3]
dk, dq = P.as_torch(keys), P.as_torch(q)
out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
pts = [list(map(int, x.split("/"))) for x in a.pts.split(",")]
idxs = {}
for pt in pts:
    K, C, mode, threads, I = pt[:5]
    hints = pt[5] if len(pt) > 5 else 3
    if (K, C) not in idxs:
        idxs[(K, C)] = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, variant=bs.KARY, k=K,
                                                                leaf_chunk=C))
    for rep in range(2):
        bs.bs_lookup_ex(idxs[(K, C)], dq, m, out, None, variant=bs.KARY, threads=threads, nreg=I,
                        kary_mode=mode, cache_hints=hints)
    torch.cuda.synchronize()
    print(json.dumps({"K": K, "C": C, "mode": mode, "threads": threads, "I": I, "hints": hints}), flush=True)
