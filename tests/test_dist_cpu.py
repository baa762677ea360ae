"""Multi-process (gloo, world_size 2 and 3) CPU tests of the PARTITIONED lookup
protocol that csrc/dist.cu runs over NCCL: route each query to the first shard
whose maximum is >= q (else the last), exchange counts, send queries, look up
locally, add the shard's global base (miss bit kept), send results back,
unroute.  The local lookup is the oracle; the protocol must reproduce the
oracle on the concatenated array — including runs of duplicates that straddle a
shard boundary (where "largest shard whose min <= q" would be wrong).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

MISS = np.uint64(1 << 63)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def route(q, shard_max):
    """dest shard = first s with shard_max[s] >= q, else P-1 (k_route_count)."""
    P = len(shard_max)
    dest = np.full(q.size, P - 1, dtype=np.int64)
    for s in range(P - 1, -1, -1):
        dest = np.where(q <= shard_max[s], s, dest)
    return dest


def protocol(rank, world, keys_global, cuts, queries_per_rank, results):
    import oracle
    lo, hi = cuts[rank], cuts[rank + 1]
    local = keys_global[lo:hi]
    q = queries_per_rank[rank]
    # build: all-gather (max, n) of every shard -> bases
    meta = [None] * world
    dist.all_gather_object(meta, (int(local[-1]), int(local.size)))
    shard_max = np.array([m[0] for m in meta], dtype=np.uint64)
    base = np.concatenate([[0], np.cumsum([m[1] for m in meta])])[:world]
    # route + counts (k_route_count / ncclAllGather of the P x P matrix)
    dest = route(q, shard_max)
    order = np.argsort(dest, kind="stable")
    perm = np.empty(q.size, dtype=np.int64)
    perm[order] = np.arange(q.size)              # slot of query i in the send buffer
    sendq = q[order]
    counts = np.bincount(dest, minlength=world)
    mat = [None] * world
    dist.all_gather_object(mat, counts.tolist())
    soff = np.concatenate([[0], np.cumsum(counts)])
    # query exchange (grouped send/recv): every rank ships segment t to rank t
    segs = [None] * world
    dist.all_gather_object(segs, [sendq[soff[t]:soff[t + 1]].tolist() for t in range(world)])
    recv = [np.array(segs[src][rank], dtype=np.uint64) for src in range(world)]
    allq = np.concatenate(recv) if recv else np.zeros(0, np.uint64)
    res = oracle.lookup(local, allq) if allq.size else np.zeros(0, np.uint64)
    res = ((res & ~MISS) + np.uint64(base[rank])) | (res & MISS)   # k_add_base
    roff = np.concatenate([[0], np.cumsum([r.size for r in recv])])
    back = [None] * world
    dist.all_gather_object(back, [res[roff[s]:roff[s + 1]].tolist() for s in range(world)])
    backres = np.concatenate([np.array(back[t][rank], dtype=np.uint64) for t in range(world)])
    out = backres[perm]                           # k_unroute
    results[rank] = out


def _worker(rank, world, port, keys_global, cuts, queries, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    protocol(rank, world, keys_global, cuts, queries, res)
    ret[rank] = res[rank].tolist()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_protocol_matches_oracle(world):
    import oracle
    rng = np.random.default_rng(world)
    n = 3000
    keys = np.sort(rng.integers(0, 900, size=n).astype(np.uint64))   # heavy duplicates
    cuts = [0] + sorted(rng.choice(np.arange(1, n), size=world - 1, replace=False).tolist()) + [n]
    # force a duplicate run across the first cut
    keys[cuts[1] - 3: cuts[1] + 3] = keys[cuts[1] - 3]
    keys = np.sort(keys)
    queries = []
    for r in range(world):
        q = np.concatenate([rng.integers(0, 1000, size=500).astype(np.uint64), keys[rng.integers(0, n, size=300)],
                            np.array([0, keys[cuts[1]], np.iinfo(np.uint64).max], dtype=np.uint64)])
        queries.append(q)
    mgr = mp.Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, keys, cuts, queries, ret), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(np.array(ret[r], dtype=np.uint64), oracle.lookup(keys, queries[r])), r


def test_min_based_routing_is_wrong_with_straddling_duplicates():
    """The tempting rule 'largest shard whose min <= q' breaks first-occurrence
    semantics when duplicates straddle a boundary; max-based routing does not."""
    keys = np.array([1, 5, 5, 5, 9], dtype=np.uint64)
    shards = [keys[:2], keys[2:]]          # the run of 5s straddles the cut
    q = np.array([5], dtype=np.uint64)
    mx = np.array([s[-1] for s in shards], dtype=np.uint64)
    assert route(q, mx)[0] == 0            # max-based: shard 0 holds the first 5
    mins = np.array([s[0] for s in shards], dtype=np.uint64)
    min_based = max(i for i in range(2) if mins[i] <= q[0])
    assert min_based == 1                  # would answer rank 2 instead of 1
