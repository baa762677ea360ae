"""bs_build_peer / bs_lookup_peer (fused peer-memory routing, include/bs.h;
SURVEY §8f f1): bit-exact vs the oracle on the concatenated array.

* world = 1: the route kernel stores every query into the rank's own window,
  the K-ary kernel's peer epilogue stores every result into its own return
  window; consecutive calls exercise the monotonic counters.
* world = 2 (one process per GPU; skipped on a one-GPU box — round 1 ran it as two processes on ONE GPU,
  which B200_PROFILING.md forbids): each process has its own window, mapped into
  the other with CUDA IPC — the same code path as two GPUs over NVLink, with a
  run of duplicates straddling the shard boundary (first-occurrence routing).
"""
import os
import socket

import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def _layout(kb, reorder=0):
    return bs.bs_layout_default(key_bytes=kb, out_bytes=8, variant=bs.KARY, reorder=reorder)


@pytest.mark.parametrize("kb", [8, 4])
def test_peer_world1(kb):
    keys = workload.gen_keys(200003, kb, seed=21)
    idx = bs.bs_build_peer(P.as_torch(keys), keys.size, _layout(kb), 0, 1, 300000)
    bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])
    out = torch.empty(300000, dtype=torch.int64, device="cuda")
    for call, (m, hr) in enumerate([(300000, 0.6), (0, 1.0), (1, 0.0), (12345, 1.0), (299999, 0.3)]):
        q = workload.gen_queries(keys, max(m, 1), seed=100 + call, hit_ratio=hr)[:m]
        dq = P.as_torch(q) if m else None
        bs.bs_lookup_peer(idx, dq, m, out)
        torch.cuda.synchronize()
        if m:
            got = P.to_numpy_unsigned(out[:m], 8)
            want = oracle.lookup(keys, q, out_bytes=8)
            assert np.array_equal(got, want), f"call {call}: first mismatch at {np.flatnonzero(got != want)[:5]}"
    # out only 8-B aligned: the finish kernel's scalar copy
    q = workload.gen_queries(keys, 4097, seed=7, hit_ratio=0.5)
    bs.bs_lookup_peer(idx, P.as_torch(q), q.size, out[1:])
    torch.cuda.synchronize()
    assert np.array_equal(P.to_numpy_unsigned(out[1:1 + q.size], 8), oracle.lookup(keys, q, out_bytes=8))
    err, calls = bs.bs_peer_status(idx)
    assert err == 0 and calls == 6
    idx.close()


@pytest.mark.parametrize("kb,n", [(8, 1), (4, 7), (8, 200003), (4, 200003), (8, 3 << 20), (4, 5 << 20)])
def test_peer_world1_bucket(kb, n):
    """layout.reorder = BUCKET: the window is partitioned and searched by the
    bucket pipeline (part.cu), whose unpartition stores every result into its
    source's return window; m spans several 8192-query tiles with ragged tails,
    one bucket (n = 200003) and several (3 / 5 Mi keys), across calls (the
    cursor re-arm and the monotonic counters)."""
    keys = workload.gen_keys(n, kb, seed=23)
    idx = bs.bs_build_peer(P.as_torch(keys), keys.size, _layout(kb, bs.REORDER_BUCKET), 0, 1, 300000)
    bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])
    out = torch.empty(300000, dtype=torch.int64, device="cuda")
    for call, (m, hr) in enumerate([(300000, 0.6), (0, 1.0), (1, 0.0), (8192, 1.0), (12345, 1.0), (299999, 0.3)]):
        q = workload.gen_queries(keys, max(m, 1), seed=200 + call, hit_ratio=hr)[:m]
        bs.bs_lookup_peer(idx, P.as_torch(q) if m else None, m, out)
        torch.cuda.synchronize()
        if m:
            got = P.to_numpy_unsigned(out[:m], 8)
            want = oracle.lookup(keys, q, out_bytes=8)
            assert np.array_equal(got, want), f"call {call}: first mismatch at {np.flatnonzero(got != want)[:5]}"
    err, calls = bs.bs_peer_status(idx)
    assert err == 0 and calls == 6
    idx.close()


def test_peer_bucket_results_window_and_overflow():
    keys = workload.gen_keys(1 << 20, 8, seed=43)
    idx = bs.bs_build_peer(P.as_torch(keys), keys.size, _layout(8, bs.REORDER_BUCKET), 0, 1, 50000)
    bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])
    q = workload.gen_queries(keys, 50000, seed=44, hit_ratio=0.5)
    bs.bs_lookup_peer(idx, P.as_torch(q), q.size, None)
    torch.cuda.synchronize()
    win = torch.as_tensor(_DeviceWindow(bs.bs_peer_results(idx), q.size), device="cuda")
    assert np.array_equal(P.to_numpy_unsigned(win, 8), oracle.lookup(keys, q, out_bytes=8))
    assert bs.bs_peer_status(idx)[0] == 0
    idx.close()
    # a window smaller than the batch: flagged, the received prefix still looked up
    idx = bs.bs_build_peer(P.as_torch(keys), keys.size, _layout(8, bs.REORDER_BUCKET), 0, 1, 20000,
                           recv_capacity=9000)
    bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])
    q = workload.gen_queries(keys, 20000, seed=45)
    out = torch.empty(20000, dtype=torch.int64, device="cuda")
    bs.bs_lookup_peer(idx, P.as_torch(q), q.size, out)
    torch.cuda.synchronize()
    assert bs.bs_peer_status(idx)[0] & 1
    idx.close()


def test_peer_overflow_flagged():
    keys = workload.gen_keys(5000, 8, seed=3)
    idx = bs.bs_build_peer(P.as_torch(keys), keys.size, _layout(8), 0, 1, 1000, recv_capacity=100)
    bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])
    q = workload.gen_queries(keys, 1000, seed=4)
    out = torch.empty(1000, dtype=torch.int64, device="cuda")
    bs.bs_lookup_peer(idx, P.as_torch(q), 1000, out)
    torch.cuda.synchronize()
    err, _ = bs.bs_peer_status(idx)
    assert err & 1
    idx.close()


def test_peer_max_m_bound_for_4byte_tags():
    """Return tags are 4 B: (src_rank << (32 - ceil(log2 world))) | src_idx, so
    max_m_local above 2^(32 - ceil(log2 world)) is rejected before any allocation."""
    keys = workload.gen_keys(1000, 8, seed=5)
    for world, limit in ((8, 1 << 29), (3, 1 << 30), (2, 1 << 31), (1, (1 << 32) - 1)):
        with pytest.raises(bs.BsError) as e:
            bs.bs_build_peer(P.as_torch(keys), keys.size, _layout(8), 0, world, limit + 1, recv_capacity=16)
        assert e.value.code == bs.BS_ERR_INVALID


def test_peer_connect_checks_order():
    a = workload.gen_keys(1000, 8, seed=5)
    lo, hi = a[:500], a[500:]
    i0 = bs.bs_build_peer(P.as_torch(hi), hi.size, _layout(8), 0, 2, 10)
    i1 = bs.bs_build_peer(P.as_torch(lo), lo.size, _layout(8), 1, 2, 10)
    with pytest.raises(bs.BsError) as e:
        bs.bs_peer_connect(i0, [bs.bs_peer_export(i0), bs.bs_peer_export(i1)])
    assert e.value.code == -6
    with pytest.raises(bs.BsError):   # rank mismatch in the blob order
        bs.bs_peer_connect(i0, [bs.bs_peer_export(i1), bs.bs_peer_export(i0)])
    with pytest.raises(bs.BsError):   # not KARY
        bs.bs_build_peer(P.as_torch(lo), lo.size, bs.bs_layout_default(key_bytes=8, out_bytes=8, variant=bs.OPT),
                         0, 1, 10)
    i0.close()
    i1.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _world2_worker(rank, world, port, keys, cut, calls, ret, kb=8, reorder=0):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)   # one process per GPU (ranks that wait on each other must not share one)
    shard = keys[:cut] if rank == 0 else keys[cut:]
    max_m = max(m for m, _ in calls)
    idx = bs.bs_build_peer(P.as_torch(shard), shard.size, _layout(kb, reorder), rank, world, max_m)
    bs.bs_peer_connect_group(idx)
    out = torch.empty(max_m, dtype=torch.int64, device="cuda")
    res = []
    for c, (m, hr) in enumerate(calls):
        q = workload.gen_queries(keys, max(m, 1), seed=1000 * rank + c, hit_ratio=hr)[:m]
        bs.bs_lookup_peer(idx, P.as_torch(q) if m else None, m, out)
        torch.cuda.synchronize()
        got = P.to_numpy_unsigned(out[:m], 8).copy()
        res.append(bool(np.array_equal(got, oracle.lookup(keys, q, out_bytes=8))))
    err, _ = bs.bs_peer_status(idx)
    dist.barrier()
    idx.close()
    ret[rank] = (res, err)
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("kb,reorder", [(8, 0), (4, 0), (8, 5), (4, 5)])
def test_peer_world2(kb, reorder):
    """World 2, one process per GPU.  Needs two GPUs: B200_PROFILING.md forbids
    running ranks whose kernels wait on each other as processes on ONE GPU
    (Xid 109 seen with 2-4 such ranks), which round 1 did; the rank logic is
    also covered on CPU (tests/test_dist_cpu.py, tests/test_bench_cpu.py)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs: peer ranks that wait on each other must not share a GPU")
    import torch.multiprocessing as mp
    keys = workload.gen_keys(300000, kb, seed=31)
    cut = 150000
    keys[cut - 3:cut + 3] = keys[cut - 3]   # duplicates straddling the boundary (still ascending)
    keys = np.sort(keys)
    calls = [(200000, 0.7), (0, 1.0), (77777, 1.0), (200000, 0.2)]
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    mp.start_processes(_world2_worker, args=(2, _free_port(), keys, cut, calls, ret, kb, reorder), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        res, err = ret[r]
        assert err == 0, f"rank {r}: peer error bits {err}"
        assert all(res), f"rank {r}: per-call parity {res}"


class _DeviceWindow:
    """Zero-copy torch view of a raw device address (CUDA array interface)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 3}


def test_peer_results_window():
    keys = workload.gen_keys(70001, 8, seed=41)
    idx = bs.bs_build_peer(P.as_torch(keys), keys.size, _layout(8), 0, 1, 50000)
    bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])
    q = workload.gen_queries(keys, 50000, seed=42, hit_ratio=0.5)
    bs.bs_lookup_peer(idx, P.as_torch(q), q.size, None)
    torch.cuda.synchronize()
    win = torch.as_tensor(_DeviceWindow(bs.bs_peer_results(idx), q.size), device="cuda")
    got = P.to_numpy_unsigned(win, 8)
    assert np.array_equal(got, oracle.lookup(keys, q, out_bytes=8))
    idx.close()


def _absent_peer_worker(rank, world, port, keys, ret):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), BS_PEER_WAIT_MS="1500")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    half = keys.size // 2
    shard = keys[:half] if rank == 0 else keys[half:]
    idx = bs.bs_build_peer(P.as_torch(shard), shard.size, _layout(8), rank, world, 1000)
    bs.bs_peer_connect_group(idx)
    if rank == 0:   # rank 1 never calls: rank 0's waits must give up, not hang the GPU
        q = workload.gen_queries(keys, 1000, seed=5)
        out = torch.empty(1000, dtype=torch.int64, device="cuda")
        bs.bs_lookup_peer(idx, P.as_torch(q), 1000, out)
        torch.cuda.synchronize()
        ret[rank] = bs.bs_peer_status(idx)[0]
    dist.barrier()
    idx.close()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_peer_absent_peer_times_out():
    import torch.multiprocessing as mp
    keys = workload.gen_keys(20000, 8, seed=81)
    mgr = mp.get_context("spawn").Manager()
    ret = mgr.dict()
    mp.start_processes(_absent_peer_worker, args=(2, _free_port(), keys, ret), nprocs=2, join=True,
                       start_method="spawn")
    assert ret[0] & 2, f"expected the timeout bit, got {ret[0]}"
