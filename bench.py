"""bench.py — lookups/s of the batched sorted-array lookup path on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  A step = one pass of the lookup path over the step's
query batch (BASELINE.json's headline workload, configs[2]: 2^26 u64 keys,
2^27 uniform random queries drawn from the key set), inputs resident in HBM.

Multi-GPU (one process per GPU): `--gpus N` without torchrun re-launches
itself under `torch.distributed.run` with N processes (127.0.0.1); under
torchrun WORLD_SIZE must equal N.  Configs and scaling:

* configs 1-4 — REPLICATED index (every rank builds the whole sorted array
  from the same deterministic generator, on its GPU), the query batch SHARDED
  across ranks: `--scaling strong` (default) splits the config's batch into N
  contiguous slices; `--scaling weak` gives every rank a batch of the config's
  size.  No collective on the data path.
* config 5 — RANGE-PARTITIONED index: rank r holds 2^30 keys drawn from its own
  value range [r*2^64/N, (r+1)*2^64/N) and 2^28 queries drawn from all shards;
  every query is routed to its owner and its result back (weak scaling).  The
  timed path is the fused peer-memory route (bs_lookup_peer); the NCCL path
  (bs_lookup_dist) is timed beside it.

Timing: W untimed warm-up steps; barrier + cuda.synchronize; CUDA events on the
launch stream around exactly K steps; max over ranks.  Inputs (queries + results
>= 2 GiB per step at the headline) exceed the 126 MB L2, so no flush.  Clocks
are sampled with nvidia-smi during the timed region.  Inputs are generated on
the GPU (workload/device.py, bit-identical to the numpy generator).

`--impl reference` times the CPU oracle (test infrastructure) on a bounded
sample of the same workload.  `--dry-run` exercises the multi-rank plumbing on
CPU (gloo) without a GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload  # noqa: E402

# name: n (per shard for config 5), key bytes, m (whole batch; per rank for config 5), hit ratio,
#       index mode, description
CONFIGS = {
    "config1": (1 << 10, 4, 1 << 16, 0.5, "replicated", "2^10 u32 keys, 2^16 uniform queries (50% hits)"),
    "config2": (1 << 20, 4, 1 << 27, 1.0, "replicated", "2^20 u32 keys (L2-resident), 2^27 uniform random queries"),
    "config3": (1 << 26, 8, 1 << 27, 1.0, "replicated", "2^26 u64 keys, 2^27 uniform random queries"),
    "config4": (1 << 30, 8, 1 << 30, 1.0, "replicated", "2^30 u64 keys replicated per GPU, 2^30 queries"),
    "config5": (1 << 30, 8, 1 << 28, 1.0, "partitioned",
                "2^30 u64 keys per GPU range-partitioned (2^33 at 8 GPUs), 2^28 queries per GPU routed to their owners"),
}
METRIC = "lookups/sec at 1/2/4/8 B200 (2^26 u64 keys, 2^27 random queries); % HBM roofline"
VARIANTS = {"naive": 0, "opt": 1, "kary": 2}
REORDER_NAMES = {0: "none", 1: "lookup", 2: "full", 3: "sorted (segment-staged)", 4: "global (2048 segments)",
                 5: "bucket (key-range partition, L2-sized buckets)"}
MISS64 = np.uint64(1 << 63)


# ----------------------------------------------------------------------------- roofline
def algorithmic_bytes_per_lookup(cfg: str, kb: int, ob: int, order: str, n: int, m_rank: int,
                                 l2_bytes: int) -> tuple[float, str]:
    """SURVEY.md §8d / DESIGN.md §6: the bytes the method must move per lookup.
    Random order, array >> L2: query in + result out + the one 32-B DRAM sector
    holding a[lb] (every level above it can be cache-resident).  Pre-sorted: the
    array is streamed once per batch.  L2-resident array (config 2): only the
    query / result stream reaches HBM.  Partitioned (config 5): + the exchange
    (query + 4-B return tag stored into the owner's window and read back, the
    8-B result stored into the source's window and read back)."""
    if order == "sorted":
        return kb + ob + n * kb / max(m_rank, 1), "key + out + n*key/m (array streamed once)"
    if n * kb <= l2_bytes // 4:
        return kb + ob, "key + out (array L2-resident; HBM carries only the query/result stream)"
    base = kb + ob + 32
    if CONFIGS[cfg][4] == "partitioned":
        return base + 2 * (kb + 4) + 2 * 8, "key + out + 32 + exchange (2 x (key + tag) + 2 x result)"
    return base, "key + out + 32 (one DRAM sector per lookup)"


def default_reorder(cfg: str, order: str) -> int:
    """The mode bench.py times by default: the key-range
    partition (BS_REORDER_BUCKET) for a random batch over an array much larger
    than L2 (for config 5: the bucket pipeline over each rank's receive window,
    bs_build_peer with layout.reorder = BUCKET), the segment-staged lookup
    (BS_REORDER_SORTED) for a sorted batch, the plain K-ary kernel otherwise
    (L2-resident arrays)."""
    n, kb, _, _, mode, _ = CONFIGS[cfg]
    if order == "sorted" and mode != "partitioned":
        return 3
    return 5 if n * kb > (256 << 20) else 0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_entry(key: str):
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        return json.load(open(tp)).get(key)
    return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region: one
    `nvidia-smi -lms 20` process streams samples from before the first timed
    launch until after the last (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, dev: int):
        self.dev = dev
        self.samples = []
        self._p = None
        self._t = None

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "20"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            # nvidia-smi can take ~1 s to emit its first line: wait for it so the
            # samples cover the timed region, then drop the pre-region ones
            t_end = time.time() + 5.0
            while not self.samples and time.time() < t_end and self._p.poll() is None:
                time.sleep(0.01)
            self.samples.clear()
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            time.sleep(0.03)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else None  # noqa: E731
        sm = [num(s[0]) for s in self.samples if num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        pw = [num(s[6]) for s in self.samples if len(s) > 6 and num(s[6]) is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------------------- ranks
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(gpus: int) -> int:
    """`--gpus N` without a launcher: run this script under torch.distributed.run
    with N processes on this node (one per GPU) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


def shard(cfg: str, scaling: str, world: int, rank: int):
    """(n keys of this rank's index, query-stream start, queries of this rank,
    queries of the whole job) for a config."""
    n, _, m, _, mode, _ = CONFIGS[cfg]
    if mode == "partitioned" or scaling == "weak":
        return n, rank * m, m, world * m
    lo, hi = m * rank // world, m * (rank + 1) // world
    return n, lo, hi - lo, m


def reduce_max(vals, world, device=None):
    """Element-wise max over ranks (float64)."""
    if world == 1:
        return list(vals)
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(vals), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


# ----------------------------------------------------------------------------- oracle legs (test infrastructure)
def cpu_baseline(keys, q, sample: int, threads: int | None = None):
    """The oracle as it stands, on the host cores, on a bounded sample."""
    import oracle
    threads = threads or len(os.sched_getaffinity(0))
    qs = q[:sample]
    t0 = time.perf_counter()
    oracle.lookup(keys, qs, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": qs.size / dt, "unit": "lookups/s", "cores": threads, "kind": "oracle",
            "sample": f"first {qs.size} queries of the same workload (C bisection, {threads} pthreads)",
            "seconds": dt}


def _gen(cfg: str, rank: int, world: int, scaling: str, order: str, device, shrink: int = 0):
    """This rank's keys and queries (torch tensors on `device`, unsigned bit
    patterns) — the same numbers on every backend (workload/device.py).
    shrink > 0 (dry runs) divides key and query counts by 2^shrink."""
    import torch
    from workload import device as wd
    n, kb, m, hr, mode, _ = CONFIGS[cfg]
    n_loc, start, m_rank, m_job = shard(cfg, scaling, world, rank)
    if shrink:
        n, n_loc = max(n >> shrink, 16), max(n_loc >> shrink, 16)
        start, m_rank, m_job = start >> shrink, max(m_rank >> shrink, world), m_job >> shrink
    if mode == "partitioned":
        span = (1 << 64) // world
        keys = wd.gen_keys_range(n_loc, rank * span, (rank + 1) * span, workload.KEY_SEED, rank, device=device)
        q = wd.gen_queries(keys, m_rank, seed=workload.QUERY_SEED, hit_ratio=hr, start=start)
        if world > 1:
            # untimed shuffle exchange: every rank's batch spans every shard
            import torch.distributed as dist
            q = q[: (q.numel() // world) * world].contiguous()
            recv = torch.empty_like(q)
            dist.all_to_all_single(recv, q)
            q = recv
        perm = torch.argsort(wd.hash_stream(workload.QUERY_SEED, 7, start, q.numel(), device))
        q = q[perm].contiguous()
        if order == "sorted":
            q = wd.sort_unsigned(q)
    else:
        keys = wd.gen_keys(n, kb, seed=workload.KEY_SEED, device=device)
        q = wd.gen_queries(keys, m_rank, seed=workload.QUERY_SEED, hit_ratio=hr, order=order, start=start)
    return keys, q, (n_loc, start, m_rank, m_job)


def make_inputs(cfg: str, order: str, rank: int = 0):
    """(keys, queries, description) as numpy arrays for tools/: this rank's inputs
    at world 1 (the whole batch), generated on the GPU when one is present."""
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    k, q, _ = _gen(cfg, rank, 1, "strong", order, dev)
    kb = CONFIGS[cfg][1]
    return _host(k, kb), _host(q, kb), CONFIGS[cfg][5]


def _host(t, kb):
    return t.cpu().numpy().view(np.uint64 if kb == 8 else np.uint32)


def run_reference(args):
    """The base contract's reference arm for this tier: the CPU oracle, as it
    stands, on the host cores, on a bounded sample of this arm's workload.
    Under torchrun only rank 0 runs."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"   # input generation only
    cfg = args.config
    n, kb, m, hr, mode, desc = CONFIGS[cfg]
    tk, tq, _ = _gen(cfg, 0, 1, args.scaling, args.order, dev)
    keys, q = _host(tk, kb), _host(tq[: args.ref_sample], kb)
    del tk, tq
    sample = min(args.ref_sample, q.size)
    for _ in range(args.warmup):
        cpu_baseline(keys, q, min(sample, 1 << 16))
    vals = [cpu_baseline(keys, q, sample) for _ in range(args.steps)]
    total_t = sum(v["seconds"] for v in vals)
    value = sample * len(vals) / total_t
    cb = dict(vals[0])
    cb["value"] = value
    cb.pop("seconds", None)
    if mode == "partitioned":
        cb["sample"] += " (over shard 0's keys)"
    line = {"metric": METRIC, "value": value, "unit": "lookups/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_t / len(vals), "higher_is_better": True,
            "scaling": "weak" if mode == "partitioned" else args.scaling, "vs_baseline": None,
            "dtype": "u64" if kb == 8 else "u32", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{cfg}: {desc}", "order": args.order,
                       "step": f"bounded sample of {sample} queries"},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- parity (test infrastructure)
def parity_replicated(keys_host, q_host, out, ob, samp_idx):
    """Sampled outputs vs the oracle (the plain lower bound + miss bit)."""
    import oracle
    import paper_2506_01576_b200 as P
    got = P.to_numpy_unsigned(out[samp_idx], ob) if hasattr(out, "device") else out[samp_idx]
    want = oracle.lookup(keys_host, q_host[samp_idx.cpu().numpy()], out_bytes=ob)
    return bool(np.array_equal(got, want))


def invariant_all(keys, q, out, ob, chunk: int = 1 << 25):
    """Every output: a[lb-1] < q <= a[lb] (a[-1] = -inf, a[n] = +inf) and the hit
    flag == (lb < n and a[lb] == q) — it determines lb uniquely.
    Verification only (torch gathers on the device, in chunks)."""
    import torch
    from workload.device import _flip
    n = keys.numel()
    u64 = keys.dtype == torch.int64
    k = _flip(keys) if u64 else keys.to(torch.int64) & 0xFFFFFFFF     # signed order == unsigned order
    for c0 in range(0, q.numel(), chunk):
        qc = q[c0:c0 + chunk]
        oc = out[c0:c0 + chunk]
        qq = _flip(qc) if u64 else qc.to(torch.int64) & 0xFFFFFFFF
        if ob == 8:
            miss = oc < 0
            lb = oc & 0x7FFFFFFFFFFFFFFF
        else:
            o = oc.to(torch.int64) & 0xFFFFFFFF
            miss = (o & 0x80000000) != 0
            lb = o & 0x7FFFFFFF
        ok = (lb >= 0) & (lb <= n)
        prev = k[(lb - 1).clamp(0, n - 1)]
        cur = k[lb.clamp(0, n - 1)]
        ok &= (lb == 0) | (prev < qq)
        ok &= (lb == n) | (qq <= cur)
        ok &= ((lb < n) & (cur == qq)) == ~miss
        if not bool(ok.all().item()):
            return False
    return True


def parity_partitioned(keys_host, q, out, world, samp_idx):
    """Sampled global results of the partitioned path vs the oracle: global
    lb(q) = sum over shards of the local lower bounds (each rank runs the oracle
    on its own shard for every rank's sampled queries), hit = any shard hits."""
    import torch
    import oracle
    qs = q[samp_idx]
    rs = out[samp_idx]
    if world > 1:
        import torch.distributed as dist
        allq = [torch.empty_like(qs) for _ in range(world)]
        allr = [torch.empty_like(rs) for _ in range(world)]
        dist.all_gather(allq, qs)
        dist.all_gather(allr, rs)
        qs, rs = torch.cat(allq), torch.cat(allr)
    qh = qs.cpu().numpy().view(np.uint64)
    loc = oracle.lookup(keys_host, qh, out_bytes=8)
    lb = (loc & ~MISS64).astype(np.int64)
    hit = ((loc & MISS64) == 0).astype(np.int64)
    t = torch.tensor(np.stack([lb, hit]), device=qs.device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    tot = t.cpu().numpy()
    want = tot[0].astype(np.uint64) | np.where(tot[1] > 0, np.uint64(0), MISS64)
    return bool(np.array_equal(rs.cpu().numpy().view(np.uint64), want))


# ----------------------------------------------------------------------------- dry run (CPU, gloo)
def run_dry(args):
    """Multi-rank plumbing without a GPU: rank/world handling, the shard plan,
    the generator on CPU at a reduced size, the oracle on each rank's slice, the
    max-over-ranks reduction and the single JSON line from rank 0."""
    import torch
    import torch.distributed as dist
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    cfg = args.config
    n, kb, m, hr, mode, desc = CONFIGS[cfg]
    n_loc, start, m_rank, m_job = shard(cfg, args.scaling, world, rank)
    # reduced problem (keys and queries / 2^16) with the same shard arithmetic and generator
    keys, q, _ = _gen(cfg, rank, world, args.scaling, args.order, "cpu", shrink=16)
    import oracle
    t0 = time.perf_counter()
    res = oracle.lookup(_host(keys, kb), _host(q, kb), out_bytes=8 if mode == "partitioned" else kb)
    dt = time.perf_counter() - t0
    ms = reduce_max([dt * 1e3], world)[0]
    per = [None] * world
    if world > 1:
        dist.all_gather_object(per, {"rank": rank, "query_start": start, "queries": m_rank, "keys": n_loc,
                                     "checksum": int(res.astype(np.uint64).sum() % (1 << 61))})
    else:
        per = [{"rank": 0, "query_start": start, "queries": m_rank, "keys": n_loc}]
    if rank == 0:
        line = {"metric": METRIC, "value": None, "unit": "lookups/s", "n_gpus": world, "steps": 0,
                "warmup": 0, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak" if mode == "partitioned" else args.scaling, "dry_run": True,
                "config": {"workload": f"{cfg}: {desc}", "queries_job": m_job}, "per_rank": per}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config3", choices=sorted(CONFIGS))
    ap.add_argument("--order", default="random", choices=["random", "sorted"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="replicated configs: strong = the config's batch split over the ranks, weak = per rank")
    ap.add_argument("--variant", default="kary", choices=sorted(VARIANTS))
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--leaf-chunk", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--nreg", type=int, default=0)
    ap.add_argument("--reorder", type=int, default=-1,
                    help="bs_reorder; -1 = the config's fastest mode: BUCKET (5) for a random batch over an "
                         "array larger than L2 (configs 3-5; config 5: the owner's lookup of its receive window), SORTED (3) for a pre-sorted batch, else NONE")
    ap.add_argument("--schedule", type=int, default=1)
    ap.add_argument("--hints", type=int, default=0x100, help="cache_hints bits; 256 = BS_HINT_AUTO (resolved at build)")
    ap.add_argument("--kary-mode", type=int, default=8,
                    help="0 warp, 1 hybrid, 2-5 tiered, 6 thread-per-lookup, 7 + flat table, 8 auto (resolved at build)")
    ap.add_argument("--no-naive", action="store_true", help="skip the naive comparison leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dist", action="store_true", help="config 5: skip the NCCL comparison path")
    ap.add_argument("--cpu-sample", type=int, default=1 << 22)
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    ap.add_argument("--dry-run", action="store_true", help="CPU-only multi-rank plumbing check (gloo)")
    ap.add_argument("--verbose", action="store_true", help="progress on stderr")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # timing rule: W >= 3
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args.gpus)
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), file=sys.stderr)
        return 2
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2506_01576_b200 as P
    from paper_2506_01576_b200 import bs

    def say(*a):
        if args.verbose:
            print(f"[rank {rank} {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    cfg = args.config
    n, kb, m_cfg, hr, mode, desc = CONFIGS[cfg]
    ob = 8 if mode == "partitioned" else kb
    if args.reorder < 0:
        args.reorder = default_reorder(cfg, args.order)
    say("generating inputs")
    dk, dq, (n_loc, qstart, m, m_job) = _gen(cfg, rank, world, args.scaling, args.order, "cuda")
    say(f"inputs: {n_loc} keys, {m} queries")
    out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[ob], device="cuda")
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size

    K = args.k or 5
    lay = bs.bs_layout_default(key_bytes=kb, out_bytes=ob, variant=VARIANTS[args.variant], k=K,
                               leaf_chunk=args.leaf_chunk, schedule=args.schedule, threads=args.threads,
                               nreg=args.nreg, reorder=args.reorder, cache_hints=args.hints,
                               kary_mode=args.kary_mode)
    stream = torch.cuda.Stream()
    dist_ms = None
    if mode == "partitioned":
        # each rank's batch holds m / world queries drawn from every shard (the
        # untimed exchange in _gen), so each rank receives ~m: a receive window
        # of m + 1/16 (an overflow would be flagged and fail the parity check)
        # instead of the never-overflowing world * m keeps the window and the
        # BUCKET workspace at ~18 GB per GPU at world 8 instead of ~73
        idx = bs.bs_build_peer(dk, n_loc, lay, rank, world, m, recv_capacity=m + m // 16 + 8192)
        if world > 1:
            bs.bs_peer_connect_group(idx)
        else:
            bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])

        def step():
            bs.bs_lookup_peer(idx, dq, m, out, stream)
    else:
        idx = bs.bs_build(dk, n_loc, lay)
        ws_bytes = bs.bs_workspace_bytes(idx, m)   # BS_REORDER_GLOBAL partitions out of place
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda") if ws_bytes else None

        def step():
            if ws is not None:
                bs.bs_lookup_ws(idx, dq, m, out, stream, ws, ws_bytes)
            else:
                bs.bs_lookup(idx, dq, m, out, stream)
    info = idx.info
    launch = bs.bs_launch_default(idx)
    say("index built", info)

    def timed(fn, steps):
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                fn()
        stream.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        c0 = bs.bs_launch_count()
        with ClockSampler(dev) as cs:
            e0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(steps):
                    fn()
            e1.record(stream)
            e1.synchronize()
        torch.cuda.synchronize()
        launches = bs.bs_launch_count() - c0
        return e0.elapsed_time(e1), cs.summary(), launches

    ms_rank, clocks, launches = timed(step, args.steps)
    say(f"timed: {ms_rank / args.steps:.3f} ms per step")
    ms = reduce_max([ms_rank], world, "cuda")[0]
    ms_step = ms / args.steps
    value = m_job * args.steps / (ms / 1e3)

    # ---- parity (every rank; test infrastructure) ----
    kh = _host(dk, kb)
    samp = torch.from_numpy(np.random.default_rng(1 + rank).integers(0, max(m, 1), size=min(m, 1 << 14))).cuda()
    if mode == "partitioned":
        peer_err = bs.bs_peer_status(idx)[0]
        parity_ok = parity_partitioned(kh, dq, out, world, samp) and peer_err == 0
        inv_ok = None
    else:
        parity_ok = parity_replicated(kh, _host(dq, kb), out, ob, samp)
        inv_ok = invariant_all(dk, dq, out, ob)
    oks = reduce_max([0.0 if parity_ok else 1.0, 0.0 if inv_ok in (True, None) else 1.0], world, "cuda")
    parity_ok, inv_ok = oks[0] == 0.0, (None if inv_ok is None else oks[1] == 0.0)

    say("parity", parity_ok, inv_ok)
    # ---- comparison legs ----
    naive_ms = None
    if not args.no_naive and args.variant != "naive" and mode == "replicated":
        def step_naive():
            bs.bs_lookup_ex(idx, dq, m, out, stream, variant=bs.NAIVE, threads=256, reorder=0)
        ns = max(1, min(args.steps, 5 if m <= (1 << 27) else 1))
        nms, _, _ = timed(step_naive, ns)
        naive_ms = reduce_max([nms / ns], world, "cuda")[0]
    if mode == "partitioned" and not args.no_dist:
        if rank == 0:
            uid = bs.bs_dist_get_uid()
        else:
            uid = None
        if world > 1:
            obj = [uid]
            torch.distributed.broadcast_object_list(obj, src=0)
            uid = obj[0]
        comm = bs.bs_dist_init(uid, rank, world)
        didx = bs.bs_build_dist(comm, dk, n_loc, bs.DIST_PARTITIONED, lay, m)
        dout = torch.empty_like(out)

        def step_dist():
            bs.bs_lookup_dist(didx, dq, m, dout, stream)
        dsteps = max(1, min(args.steps, 5))
        dms, _, _ = timed(step_dist, dsteps)
        dist_ms = reduce_max([dms / dsteps], world, "cuda")[0]
        dist_ok = parity_partitioned(kh, dq, dout, world, samp)
        didx.close()
        bs.bs_dist_destroy(comm)
        del dout
    else:
        dist_ok = None

    # ---- end to end through the public API, host buffers ----
    e2e = None
    if not args.no_e2e:
        hq = dq.cpu().pin_memory()
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        e2e_steps = max(1, min(args.steps, 3))
        if mode == "partitioned":
            # bs_lookup_peer is device-to-device; the user's host round trip is
            # H2D of the queries, the call, D2H of the results on the same stream
            def e2e_step():
                with torch.cuda.stream(stream):
                    dq.copy_(hq, non_blocking=True)
                    bs.bs_lookup_peer(idx, dq, m, out, stream)
                    hout.copy_(out, non_blocking=True)
                stream.synchronize()
            api = "H2D copy + bs_lookup_peer + D2H copy (pinned host buffers)"
        else:
            def e2e_step():
                bs.bs_lookup_host(idx, hq, m, hout, stream)
            api = ("bs_lookup_host (pinned host buffers; chunks of 2^22 queries overlap the PCIe copies, "
                   "each chunk in the in-place mode: the out-of-place reorderings need a caller workspace)")
        e2e_step()   # warm (allocates staging)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        dt = reduce_max([(time.perf_counter() - t0) / e2e_steps], world, "cuda")[0]
        # the PCIe floor of the same bytes: the step's H2D and D2H copies alone,
        # concurrently on two streams (the link is full duplex), no lookup
        s2 = torch.cuda.Stream()

        def copies():
            with torch.cuda.stream(stream):
                dq.copy_(hq, non_blocking=True)   # same values: dq is hq's source
            with torch.cuda.stream(s2):
                hout.copy_(out, non_blocking=True)
            stream.synchronize()
            s2.synchronize()
        copies()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            copies()
        dcp = reduce_max([(time.perf_counter() - t0) / e2e_steps], world, "cuda")[0]
        e2e = {"value": m_job / dt, "unit": "lookups/s", "h2d_bytes_per_step": m * kb,
               "d2h_bytes_per_step": m * ob, "ms_per_step": dt * 1e3, "api": api,
               "pcie_floor_ms": dcp * 1e3, "frac_of_pcie_floor": dcp / dt}
        del hq, hout

    # ---- roofline ----
    peak, peak_src = peaks()
    bpl, bpl_why = algorithmic_bytes_per_lookup(cfg, kb, ob, args.order, n_loc, m, l2_bytes)
    achieved = bpl * m / (ms_step / 1e3) / 1e9          # per GPU (max-over-ranks time)
    tkey = (f"{cfg}/{args.order}/{args.variant}/K{info['k']}/C{info['leaf_chunk']}/mode{launch.kary_mode}"
            + ("/peer" if mode == "partitioned" else "") + (f"/r{launch.reorder}" if launch.reorder else ""))
    te = traffic_entry(tkey)
    traffic = None
    if te and te.get("queries") == m:
        traffic = te["dram_bytes_per_launch"]
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu --set full)",
            "traffic_GBps": traffic / (ms_step / 1e3) / 1e9 if traffic else None,
            "traffic_frac": traffic / (ms_step / 1e3) / 1e9 / peak if traffic else None,
            "traffic_key": tkey, "alg_bytes_per_launch": bpl * m, "bytes_per_lookup_alg": bpl,
            "bytes_per_lookup_model": bpl_why, "peak_source": peak_src, "per": "GPU"}
    if bpl_why.startswith("key + out (array L2") and te and te.get("l2_read_sectors_per_lookup"):
        # the binding roof of an L2-resident array is the L2: sectors the
        # kernel reads (ncu) at this run's speed vs the measured random-sector L2 rate
        lp = os.path.join(ROOT, "profiles", "l2_peak.json")
        if os.path.exists(lp):
            l2 = json.load(open(lp))
            ach = te["l2_read_sectors_per_lookup"] * 32 * m / (ms_step / 1e3) / 1e9
            pk = l2["l2_read_GBps_random_32B_sectors"]
            roof["l2"] = {"bound": "l2", "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk,
                          "sectors_per_lookup": te["l2_read_sectors_per_lookup"],
                          "peak_source": "measured (profiles/l2_peak.json, random 32-B sectors from an L2-resident buffer)"}
    if te and te.get("kernels"):
        # a step of several kernels: the roofline is the step's (sum of its launches); shares beside it
        roof["kernels"] = [{"kernel": k["kernel"], "share_ncu": k["ms"] / te["ncu_ms"],
                            "dram_B_per_lookup": k["dram_B_per_lookup"]} for k in te["kernels"]]
        roof["traffic_per_lookup"] = te["dram_bytes_per_lookup"]

    line = {
        "metric": METRIC, "value": value, "unit": "lookups/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if mode == "partitioned" else args.scaling,
        "vs_baseline": None, "dtype": "u64" if kb == 8 else "u32", "data": "synthetic (workload/device.py, seeded)",
        "config": {"workload": f"{cfg}: {desc}", "order": args.order, "variant": args.variant,
                   "index": mode, "k": info["k"], "leaf_chunk": info["leaf_chunk"],
                   "kary_levels": info["kary_levels"], "kary_smem_levels": info["kary_smem_levels"],
                   "keys_per_gpu": n_loc, "queries_per_gpu": m, "queries_job": m_job,
                   "cache_hints": launch.cache_hints, "kary_mode": launch.kary_mode,
                   "reorder": REORDER_NAMES.get(launch.reorder, str(launch.reorder)),
                   "parallelism": (f"{mode} x{world}" if world > 1 else "1 GPU"),
                   "l2": ("inputs larger than L2 (queries + results per step > 126 MB), no flush"
                          if m * (kb + ob) > 2 * l2_bytes else "inputs smaller than L2, no flush")},
        "roofline": roof,
        "gpu_launches": int(reduce_max([launches], world, "cuda")[0]),
        "clocks": clocks,
        "parity_sample_ok": parity_ok,
        "invariant_all_ok": inv_ok,
        "per_rank_ms_per_step_max": ms_step,
    }
    if naive_ms:
        line["naive_ms_per_step"] = naive_ms
        line["speedup_vs_naive"] = naive_ms / ms_step
    if dist_ms:
        line["nccl_path"] = {"api": "bs_lookup_dist", "ms_per_step": dist_ms, "value": m_job / (dist_ms / 1e3),
                             "parity_sample_ok": dist_ok}
    if e2e:
        line["e2e"] = e2e
    if rank == 0:
        line["cpu_baseline"] = cpu_baseline(kh, _host(dq[: args.cpu_sample], kb), args.cpu_sample)
        line["cpu_baseline"].pop("seconds", None)
        if mode == "partitioned":
            line["cpu_baseline"]["sample"] += " (over this rank's shard)"
        print(json.dumps(line), flush=True)
    idx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
