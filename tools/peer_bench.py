"""Routing overhead of the PARTITIONED paths on ONE GPU (world = 1): the same
config-3 workload through bs_lookup (no routing), bs_lookup_dist (NCCL:
route/count/host-sync/all-to-all/unroute) and bs_lookup_peer (fused peer
stores + device counters).  CUDA events on the launch stream, median of
--reps (max over ranks); one JSON line per path.  Under torchrun (world > 1, one process per
GPU) every rank holds 2^26/world keys and 2^27/world queries (partitioned);
ranks beyond the visible GPUs share them (functional check only, e.g.
`torchrun --nproc-per-node 2` on a 1-GPU box).

python tools/peer_bench.py [--reps 10] [--m-log2 27] [--n-log2 26]
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

import workload  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def timed(fn, reps, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--m-log2", type=int, default=27)
    ap.add_argument("--n-log2", type=int, default=26)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # ranks beyond the visible GPUs share them (functional runs on a 1-GPU box)
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    n, m = 1 << a.n_log2, (1 << a.m_log2) // world
    keys = workload.gen_keys(n, 8, seed=workload.KEY_SEED)
    cut = [n * r // world for r in range(world + 1)]
    shard = keys[cut[rank]:cut[rank + 1]]
    q = workload.gen_queries(keys, m, seed=workload.QUERY_SEED, start=rank * m)
    dq = P.as_torch(q)
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    lay = bs.bs_layout_default(key_bytes=8, out_bytes=8, variant=bs.KARY)
    rows = []
    if world == 1:
        idx = bs.bs_build(P.as_torch(keys), n, lay)
        rows.append(("bs_lookup", timed(lambda: bs.bs_lookup(idx, dq, m, out, s), a.reps, s)))
        idx.close()
        uid = bs.bs_dist_get_uid()
        comm = bs.bs_dist_init(uid, 0, 1)
        idx = bs.bs_build_dist(comm, P.as_torch(keys), n, bs.DIST_PARTITIONED, lay, m)
        rows.append(("bs_lookup_dist (NCCL)", timed(lambda: bs.bs_lookup_dist(idx, dq, m, out, s), a.reps, s)))
        idx.close()
        bs.bs_dist_destroy(comm)
    pidx = bs.bs_build_peer(P.as_torch(shard), shard.size, lay, rank, world, m)
    if world > 1:
        bs.bs_peer_connect_group(pidx)
    else:
        bs.bs_peer_connect(pidx, [bs.bs_peer_export(pidx)])
    rows.append(("bs_lookup_peer (fused, results left in the return window)",
                 timed(lambda: bs.bs_lookup_peer(pidx, dq, m, None, s), a.reps, s)))
    rows.append(("bs_lookup_peer (fused)", timed(lambda: bs.bs_lookup_peer(pidx, dq, m, out, s), a.reps, s)))
    err, _ = bs.bs_peer_status(pidx)
    import oracle
    sample = np.arange(0, m, max(1, m // 4096))
    got = P.to_numpy_unsigned(out, 8)[sample]
    ok = bool(np.array_equal(got, oracle.lookup(keys, q[sample], out_bytes=8))) and err == 0
    if world > 1:   # the job's time is the slowest rank's
        import torch.distributed as dist
        t = torch.tensor([ms for _, ms in rows] + [0.0 if ok else 1.0], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rows = [(name, float(t[i])) for i, (name, _) in enumerate(rows)]
        ok = ok and float(t[-1]) == 0.0
    if rank == 0:
        for name, ms in rows:
            print(json.dumps({"path": name, "world": world, "n": n, "m_per_rank": m, "ms": ms,
                              "G_lookups_per_s": world * m / ms / 1e6, "parity_sample_ok": ok}))
    pidx.close()


if __name__ == "__main__":
    main()
