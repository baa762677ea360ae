"""Per-call cost of a small lookup batch (config 1: 2^10 u32 keys, 2^16
queries): host time per bs_lookup call (wall clock over N back-to-back calls,
no sync between them) and device time per call (CUDA events over the same N
calls).  A device time that equals the host time means the GPU waits on the
host (launch-bound), not on the kernel.

python tools/host_overhead.py
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_01576_b200 as P  # noqa: E402
import workload  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def main():
    torch.cuda.set_device(0)
    keys = workload.gen_keys(1 << 10, 4)
    q = workload.gen_queries(keys, 1 << 16, hit_ratio=0.5)
    dk, dq = P.as_torch(keys), P.as_torch(q)
    out = torch.empty(q.size, dtype=torch.int32, device="cuda")
    idx = bs.bs_build(dk, keys.size, bs.bs_layout_default(key_bytes=4, out_bytes=4))
    s = torch.cuda.Stream()
    N = 2000
    for _ in range(50):
        bs.bs_lookup(idx, dq, q.size, out, s)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    for _ in range(N):
        bs.bs_lookup(idx, dq, q.size, out, s)
    t1 = time.perf_counter()
    e1.record(s)
    e1.synchronize()
    print(json.dumps({"calls": N, "host_us_per_call": (t1 - t0) / N * 1e6,
                      "device_us_per_call": e0.elapsed_time(e1) / N * 1e3}), flush=True)
    idx.close()


if __name__ == "__main__":
    main()
