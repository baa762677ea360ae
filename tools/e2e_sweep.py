"""bs_lookup_host pipeline sweep: stages x chunk size, plus raw PCIe copy rates.

Each point runs in a fresh index (the knobs are read when the host context is
created).  Prints one JSON line per point.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402

torch.cuda.set_device(0)
keys, q, _ = bench.make_inputs("config3", "random", 0)
n, kb, m = bench.CONFIGS["config3"][:3]
dk = P.as_torch(keys)
hq = torch.from_numpy(q.view(np.int64)).pin_memory()
hout = torch.empty(m, dtype=torch.int64).pin_memory()
dbuf = torch.empty(m, dtype=torch.int64, device="cuda")
for name, fn in (("h2d", lambda: dbuf.copy_(hq, non_blocking=True)), ("d2h", lambda: hout.copy_(dbuf, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(json.dumps({"copy": name, "GBps": m * 8 / dt / 1e9}), flush=True)
del dbuf
for stages in (2, 3, 4, 6, 8):
    for lg in (20, 22, 24):
        os.environ["BS_HOST_STAGES"] = str(stages)
        os.environ["BS_HOST_CHUNK_LOG2"] = str(lg)
        idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=8, out_bytes=8))
        bs.bs_lookup_host(idx, hq, m, hout)
        t0 = time.perf_counter()
        for _ in range(3):
            bs.bs_lookup_host(idx, hq, m, hout)
        dt = (time.perf_counter() - t0) / 3
        print(json.dumps({"stages": stages, "chunk_log2": lg, "ms": dt * 1e3, "G_lookups_per_s": m / dt / 1e9}), flush=True)
        idx.close()
