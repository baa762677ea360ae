"""bench.py — lookups/s of the batched sorted-array lookup path on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  A step = one bs_lookup over the whole query batch of
BASELINE.json's headline workload (configs[2]: 2^26 u64 keys, 2^27 uniform
random queries drawn from the key set), inputs resident in HBM.  N > 1
(torchrun, one process per GPU): REPLICATED mode — every rank holds the whole
index and its own 2^27-query shard; no collective on the data path; weak
scaling.  `--impl reference` times the CPU oracle (test infrastructure) on a
bounded sample of the same workload.

Timing: W untimed warm-up steps; barrier + cuda.synchronize; CUDA events on
the launch stream around exactly K steps; max over ranks.  Inputs (1 GiB of
queries + 1 GiB of results per step) are larger than the 126 MB L2, so no
explicit flush.  Clocks are sampled with nvidia-smi during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload  # noqa: E402

CONFIGS = {
    # name: (n, key_bytes, m, hit_ratio, description)
    "config1": (1 << 10, 4, 1 << 16, 0.5, "2^10 u32 keys, 2^16 uniform queries (50% hits)"),
    "config2": (1 << 20, 4, 1 << 27, 1.0, "2^20 u32 keys (L2-resident), 2^27 uniform random queries"),
    "config3": (1 << 26, 8, 1 << 27, 1.0, "2^26 u64 keys, 2^27 uniform random queries"),
    "config4": (1 << 30, 8, 1 << 27, 1.0, "2^30 u64 keys replicated, 2^27 queries per GPU"),
}
METRIC = "lookups/sec at 1/2/4/8 B200 (2^26 u64 keys, 2^27 random queries); % HBM roofline"
VARIANTS = {"naive": 0, "opt": 1, "kary": 2}


def algorithmic_bytes_per_lookup(kb: int, ob: int, order: str, n: int, m: int) -> float:
    """query in + result out + the one DRAM sector that holds
    a[lb] (random order, array >> L2); pre-sorted order streams the array once."""
    if order == "sorted":
        return kb + ob + n * kb / m
    return kb + ob + 32


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md)"


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


def make_inputs(cfg: str, order: str, rank: int):
    n, kb, m, hr, desc = CONFIGS[cfg]
    keys = workload.gen_keys(n, kb, seed=workload.KEY_SEED)
    q = workload.gen_queries(keys, m, seed=workload.QUERY_SEED, hit_ratio=hr, order=order, start=rank * m)
    return keys, q, desc


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


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    keys, q, desc = make_inputs(args.config, args.order, 0)
    sample = args.ref_sample
    for _ in range(args.warmup):
        cpu_baseline(keys, q, min(sample, 1 << 16))
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_baseline(keys, q, sample))
    total_t = sum(v["seconds"] for v in vals)
    value = sample * len(vals) / total_t
    cb = dict(vals[0])
    cb["value"] = value
    cb.pop("seconds", None)
    line = {"metric": METRIC, "value": value, "unit": "lookups/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_t / len(vals), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": CONFIGS[args.config][1] == 8 and "u64" or "u32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: {desc}", "order": args.order,
                       "step": f"bounded sample of {sample} queries"},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config3", choices=sorted(CONFIGS))
    ap.add_argument("--order", default="random", choices=["random", "sorted"])
    ap.add_argument("--variant", default="kary", choices=sorted(VARIANTS))
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--leaf-chunk", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--nreg", type=int, default=0)
    ap.add_argument("--reorder", type=int, default=0)
    ap.add_argument("--schedule", type=int, default=1)
    ap.add_argument("--hints", type=int, default=0x100, help="cache_hints bits; 256 = BS_HINT_AUTO (resolved at build)")
    ap.add_argument("--kary-mode", type=int, default=8,
                    help="0 warp, 1 hybrid, 2-5 tiered, 6 thread-per-lookup, 7 + flat table, 8 auto (resolved at build)")
    ap.add_argument("--no-naive", action="store_true", help="skip the naive comparison leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 22)
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # timing rule: W >= 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2506_01576_b200 as P
    from paper_2506_01576_b200 import bs

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    keys, q, desc = make_inputs(args.config, args.order, rank)
    n, kb, m, hr, _ = CONFIGS[args.config]
    ob = kb
    dk = P.as_torch(keys)
    dq = P.as_torch(q)
    out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[ob], device="cuda")

    K = args.k or 5
    C = args.leaf_chunk   # 0 = auto (resolved at build; config 3 -> 16)
    lay = bs.bs_layout_default(key_bytes=kb, out_bytes=ob, variant=VARIANTS[args.variant], k=K, leaf_chunk=C,
                               schedule=args.schedule, threads=args.threads, nreg=args.nreg,
                               reorder=args.reorder, cache_hints=args.hints,
                               kary_mode=args.kary_mode)
    idx = bs.bs_build(dk, n, lay)
    C = idx.info["leaf_chunk"]
    del dk
    stream = torch.cuda.Stream()

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
        with ClockSampler(dev) as cs:
            e0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(steps):
                    fn()
            e1.record(stream)
            e1.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, cs.summary()

    def step():
        bs.bs_lookup(idx, dq, m, out, stream)

    ms, clocks = timed(step, args.steps)
    ms_step = ms / args.steps
    value = world * m * args.steps / (ms / 1e3)

    # parity spot check: sampled outputs vs the oracle, every run
    import oracle
    samp = np.random.default_rng(1).integers(0, m, size=1 << 14)
    got = P.to_numpy_unsigned(out, ob)[samp]
    want = oracle.lookup(keys, q[samp], out_bytes=ob)
    parity_ok = bool(np.array_equal(got, want))

    # naive Listing-1 baseline on the same inputs (the >= 2x target)
    naive_ms = None
    if not args.no_naive and args.variant != "naive":
        def step_naive():
            bs.bs_lookup_ex(idx, dq, m, out, stream, variant=bs.NAIVE, threads=256)
        nms, _ = timed(step_naive, max(1, min(args.steps, 5)))
        naive_ms = nms / max(1, min(args.steps, 5))

    # end to end through the C ABI from pinned host memory
    e2e = None
    if not args.no_e2e:
        hq = torch.from_numpy(q.view({4: np.int32, 8: np.int64}[kb])).pin_memory()
        hout = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[ob]).pin_memory()
        bs.bs_lookup_host(idx, hq, m, hout, stream)   # warm (allocates staging)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            bs.bs_lookup_host(idx, hq, m, hout, stream)
        dt = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([dt], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": world * m / dt, "unit": "lookups/s", "h2d_bytes_per_step": m * kb,
               "d2h_bytes_per_step": m * ob, "ms_per_step": dt * 1e3, "api": "bs_lookup_host (pinned host buffers)"}

    peak, peak_src = peaks()
    bpl = algorithmic_bytes_per_lookup(kb, ob, args.order, n, m)
    achieved = bpl * m / (ms_step / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        key = f"{args.config}/{args.order}/{args.variant}/K{K}/C{C}/mode{bs.bs_launch_default(idx).kary_mode}"
        if key in tj:
            traffic = tj[key]["dram_bytes_per_launch"]
    info = idx.info
    line = {
        "metric": METRIC, "value": value, "unit": "lookups/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64" if kb == 8 else "u32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {desc}", "order": args.order, "variant": args.variant,
                   "k": info["k"], "leaf_chunk": info["leaf_chunk"], "kary_levels": info["kary_levels"],
                   "kary_smem_levels": info["kary_smem_levels"], "queries_per_gpu": m,
                   "cache_hints": bs.bs_launch_default(idx).cache_hints,
                   "kary_mode": bs.bs_launch_default(idx).kary_mode,
                   "parallelism": f"replicated x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2 (queries+results 2 GiB per step > 126 MB), no flush"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu --set full)",
                     # SURVEY §8d metric (2): the bytes actually touched (ncu) at this run's speed
                     "traffic_GBps": traffic / (ms_step / 1e3) / 1e9 if traffic else None,
                     "traffic_frac": traffic / (ms_step / 1e3) / 1e9 / peak if traffic else None,
                     "alg_bytes_per_launch": bpl * m, "bytes_per_lookup_alg": bpl, "peak_source": peak_src},
        "gpu_launches": args.steps,
        "clocks": clocks,
        "parity_sample_ok": parity_ok,
    }
    if naive_ms:
        line["naive_ms_per_step"] = naive_ms
        line["speedup_vs_naive"] = naive_ms / ms_step
    if e2e:
        line["e2e"] = e2e
    if rank == 0:
        n_cpu = args.cpu_sample
        line["cpu_baseline"] = cpu_baseline(keys, q, n_cpu)
        line["cpu_baseline"].pop("seconds", None)
        print(json.dumps(line))
    idx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
