"""Minimal driver for ncu: build one index and launch one variant a few times.

ncu --set full -k regex:k_kary -s 2 -c 1 -o gpurun_out/kary python tools/one_launch.py --variant kary
"""
from __future__ import annotations

import argparse
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
ap.add_argument("--variant", default="kary")
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--k", type=int, default=17)
ap.add_argument("--c", type=int, default=16)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--nreg", type=int, default=0)
ap.add_argument("--reorder", type=int, default=0)
ap.add_argument("--sched", type=int, default=1)
ap.add_argument("--pin", type=int, default=1)
ap.add_argument("--hints", type=int, default=3)
ap.add_argument("--l2fetch", type=int, default=0)
ap.add_argument("--mode", type=int, default=1, help="kary_mode: 1 hybrid, 0 warp-cooperative")
a = ap.parse_args()
torch.cuda.set_device(0)
if a.l2fetch:
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaFree(None)
    print("cudaDeviceSetLimit(L2 fetch) rc", rt.cudaDeviceSetLimit(ctypes.c_int(0x05), ctypes.c_size_t(a.l2fetch)))
keys, q, _ = bench.make_inputs(a.config, a.order, 0)
n, kb, m = bench.CONFIGS[a.config][:3]
v = bench.VARIANTS[a.variant]
idx = bs.bs_build(P.as_torch(keys), n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb, variant=v, k=a.k,
                                                            leaf_chunk=a.c))
dq = P.as_torch(q)
out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
for _ in range(a.launches):
    bs.bs_lookup_ex(idx, dq, m, out, None, variant=v, threads=a.threads, nreg=a.nreg, reorder=a.reorder,
                    schedule=a.sched, use_pinned=a.pin, cache_hints=a.hints, kary_mode=a.mode)
torch.cuda.synchronize()
print("done", idx.info)
