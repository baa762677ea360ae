"""bench.py's multi-rank plumbing on CPU (no GPU): self-launch of N ranks,
WORLD_SIZE checks, the shard plan, and the partitioned-mode parity check
(global lb = sum of the shards' oracle lower bounds) under gloo, world 2."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       env=e, timeout=600, cwd=ROOT)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return r.returncode, lines, r.stderr


@pytest.mark.parametrize("cfg,scaling", [("config3", "strong"), ("config4", "weak"), ("config5", "strong")])
def test_bench_self_launches_two_ranks(cfg, scaling):
    rc, lines, err = _run(["--gpus", "2", "--dry-run", "--config", cfg, "--scaling", scaling])
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, "exactly one JSON line (rank 0)"
    line = lines[0]
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    per = sorted(line["per_rank"], key=lambda d: d["rank"])
    assert [d["rank"] for d in per] == [0, 1]
    n, kb, m, hr, mode, _ = bench.CONFIGS[cfg]
    if mode == "partitioned":
        assert line["scaling"] == "weak"
        assert all(d["queries"] == m and d["keys"] == n for d in per)
        assert line["config"]["queries_job"] == 2 * m
    elif scaling == "strong":
        # contiguous slices that tile the config's batch
        assert per[0]["query_start"] == 0 and per[1]["query_start"] == per[0]["queries"]
        assert per[0]["queries"] + per[1]["queries"] == m == line["config"]["queries_job"]
    else:
        assert all(d["queries"] == m for d in per) and per[1]["query_start"] == m


def test_bench_world_mismatch_fails():
    rc, lines, err = _run(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert rc == 2 and not lines


def test_shard_plan_strong_covers_batch():
    for world in (1, 2, 3, 4, 8):
        got = [bench.shard("config3", "strong", world, r) for r in range(world)]
        starts = [g[1] for g in got]
        sizes = [g[2] for g in got]
        assert starts[0] == 0 and sum(sizes) == 1 << 27
        assert all(starts[i] + sizes[i] == starts[i + 1] for i in range(world - 1))
        assert all(g[3] == 1 << 27 for g in got)


def test_algorithmic_bytes_models():
    l2 = 126 << 20
    assert bench.algorithmic_bytes_per_lookup("config3", 8, 8, "random", 1 << 26, 1 << 27, l2)[0] == 48
    assert bench.algorithmic_bytes_per_lookup("config3", 8, 8, "sorted", 1 << 26, 1 << 27, l2)[0] == 20
    assert bench.algorithmic_bytes_per_lookup("config2", 4, 4, "random", 1 << 20, 1 << 27, l2)[0] == 8
    assert bench.algorithmic_bytes_per_lookup("config4", 8, 8, "random", 1 << 30, 1 << 30, l2)[0] == 48
    assert bench.algorithmic_bytes_per_lookup("config5", 8, 8, "random", 1 << 30, 1 << 28, l2)[0] == 48 + 24 + 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _parity_worker(rank, world, port, keys_global, cuts, qs, want, bad):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local = keys_global[cuts[rank]:cuts[rank + 1]]
    q = torch.from_numpy(qs[rank].view(np.int64))
    out = torch.from_numpy(want[rank].view(np.int64).copy())
    samp = torch.arange(q.numel())
    ok = bench.parity_partitioned(local, q, out, world, samp)
    if rank == 1:
        out[bad] ^= 1        # one wrong result on one rank must be seen by every rank
    ok_bad = bench.parity_partitioned(local, q, out, world, samp)
    assert ok and not ok_bad, (rank, ok, ok_bad)
    dist.destroy_process_group()


def test_parity_partitioned_gloo_world2():
    import oracle
    import workload
    rng = np.random.default_rng(3)
    keys = np.sort(np.concatenate([workload.gen_keys(3000, 8, seed=4), np.full(7, 1 << 40, dtype=np.uint64)]))
    cut = int(np.searchsorted(keys, np.uint64(1 << 40))) + 3      # duplicates straddle the cut
    cuts = [0, cut, keys.size]
    qs = [np.concatenate([rng.choice(keys, 500), rng.integers(0, 1 << 63, 100, dtype=np.uint64),
                          np.array([0, (1 << 64) - 1, 1 << 40], dtype=np.uint64)]) for _ in range(2)]
    want = [oracle.lookup(keys, q, out_bytes=8) for q in qs]
    mp.spawn(_parity_worker, args=(2, _free_port(), keys, cuts, qs, want, 17), nprocs=2, join=True)


def test_default_reorder_per_config():
    """bench.py times the config's fastest mode by default: the
    key-range partition for random batches over arrays larger than L2, the
    segment-staged lookup for pre-sorted batches, the plain kernels otherwise."""
    import bench
    assert bench.default_reorder("config3", "random") == 5
    assert bench.default_reorder("config4", "random") == 5
    assert bench.default_reorder("config3", "sorted") == 3
    assert bench.default_reorder("config2", "random") == 0
    assert bench.default_reorder("config1", "random") == 0
    assert bench.default_reorder("config5", "random") == 5
