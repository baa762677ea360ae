"""Small end-to-end run of every lookup mode, each case checked against the
oracle (a quick all-modes parity pass; compute-sanitizer is closed on the GPU
pool, so bad accesses are hunted with small cases like these, bounds checks
and the oracle).

python tools/all_modes_run.py
Cases: the K-ary default, OPT, naive, SORTED, GLOBAL, BUCKET fine (u32 / u64,
both output widths, ragged batch) and two-level (BS_BUCKET_TWO=1 at build),
bs_lookup_peer at world 1 (K-ary epilogue and the bucket pipeline), merge.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
import workload  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402

OTYPE = {4: torch.int32, 8: torch.int64}


def check(name, keys, q, out, ob):
    torch.cuda.synchronize()
    got = P.to_numpy_unsigned(out[:q.size], ob)
    want = oracle.lookup(keys, q, out_bytes=ob)
    ok = bool(np.array_equal(got, want))
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def plain(kb, ob, n, m, name, reorder=0, order="random", **launch):
    keys = workload.gen_keys(n, kb, seed=n + kb)
    q = workload.gen_queries(keys, m, seed=m + ob, hit_ratio=0.5)
    if order == "sorted":
        q = np.sort(q)
    idx = bs.bs_build(P.as_torch(keys), n, bs.bs_layout_default(key_bytes=kb, out_bytes=ob))
    out = torch.empty(m, dtype=OTYPE[ob], device="cuda")
    dq = P.as_torch(q)
    if reorder in (4, 5):
        nb = bs.bs_workspace_bytes(idx, m, reorder=reorder)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        bs.bs_lookup_ws(idx, dq, m, out, None, ws, nb, reorder=reorder, **launch)
    else:
        bs.bs_lookup_ex(idx, dq, m, out, None, reorder=reorder, **launch)
    ok = check(name, keys, q, out, ob)
    idx.close()
    return ok


def peer(kb, n, m, reorder, name):
    keys = workload.gen_keys(n, kb, seed=7 * n + kb)
    lay = bs.bs_layout_default(key_bytes=kb, out_bytes=8, variant=bs.KARY, reorder=reorder)
    idx = bs.bs_build_peer(P.as_torch(keys), n, lay, 0, 1, m)
    bs.bs_peer_connect(idx, [bs.bs_peer_export(idx)])
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    ok = True
    for c, mm in enumerate((m, m // 3 + 1)):
        q = workload.gen_queries(keys, mm, seed=c, hit_ratio=0.6)
        bs.bs_lookup_peer(idx, P.as_torch(q), mm, out)
        ok &= check(f"{name} call {c}", keys, q, out, 8)
    err, _ = bs.bs_peer_status(idx)
    ok &= err == 0
    idx.close()
    return ok


def merge(kb):
    keys = workload.gen_keys(100003, kb, seed=3)
    ins = workload.gen_keys(5001, kb, seed=4)
    idx = bs.bs_build(P.as_torch(keys), keys.size, bs.bs_layout_default(key_bytes=kb, out_bytes=8))
    nidx = bs.bs_merge(idx, P.as_torch(ins), ins.size)
    allk = np.sort(np.concatenate([keys, ins]))
    q = workload.gen_queries(allk, 20000, seed=5)
    out = torch.empty(q.size, dtype=torch.int64, device="cuda")
    bs.bs_lookup(nidx, P.as_torch(q), q.size, out)
    ok = check(f"merge u{8 * kb}", allk, q, out, 8)
    idx.close()
    nidx.close()
    return ok


def main():
    torch.cuda.set_device(0)
    ok = True
    for kb in (8, 4):
        ok &= plain(kb, kb, 300007, 50001, f"kary u{8 * kb}")
        ok &= plain(kb, 8, 300007, 20011, f"opt u{8 * kb}", variant=bs.OPT)
        ok &= plain(kb, 8, 300007, 20011, f"naive u{8 * kb}", variant=bs.NAIVE)
        ok &= plain(kb, 8, 300007, 50001, f"sorted u{8 * kb}", reorder=3, order="sorted")
        ok &= plain(kb, 8, 300007, 50001, f"global u{8 * kb}", reorder=4)
        for ob in (8, 4):
            ok &= plain(kb, ob, 300007, 50001, f"bucket fine u{8 * kb} ob{ob}", reorder=5)
    os.environ["BS_BUCKET_TWO"] = "1"
    for kb in (8, 4):
        ok &= plain(kb, 8, (5 << 20) + 3, 40009, f"bucket two-level u{8 * kb}", reorder=5)
    del os.environ["BS_BUCKET_TWO"]
    for kb in (8, 4):
        ok &= peer(kb, 300007, 30001, 0, f"peer kary u{8 * kb}")
        ok &= peer(kb, 300007, 30001, 5, f"peer bucket u{8 * kb}")
    ok &= merge(8)
    print("ALL OK" if ok else "FAILURES", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
