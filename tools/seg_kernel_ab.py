"""BS_REORDER_SORTED: the image-tree kernel vs the bracketed-bisection kernel
(BS_SEG_KERNEL) over key width and queries per key, sorted batches, one B200.

python tools/seg_kernel_ab.py > gpurun_out/seg_kernel_ab.jsonl
Each point: median of 5 launches (CUDA events) after 2 warm-ups, checked on a
2^12 sample against the oracle.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2506_01576_b200 as P  # noqa: E402
import workload.device as wd  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402
from tools.bucket_sweep import time_launch  # noqa: E402


def main():
    torch.cuda.set_device(0)
    m = 1 << 27
    for kb in (8, 4):
        for lg in (20, 23, 24, 26):
            n = 1 << lg
            dk = wd.gen_keys(n, kb, device="cuda")
            dq = wd.gen_queries(dk, m, order="sorted")
            out = torch.empty(m, dtype={4: torch.int32, 8: torch.int64}[kb], device="cuda")
            keys = P.to_numpy_unsigned(dk, kb)
            samp = np.random.default_rng(lg).integers(0, m, size=1 << 12)
            want = oracle.lookup(keys, P.to_numpy_unsigned(dq[torch.from_numpy(samp).cuda()], kb), out_bytes=kb)
            idx = bs.bs_build(dk, n, bs.bs_layout_default(key_bytes=kb, out_bytes=kb))
            for kern in ("eytz", "bracket"):
                os.environ["BS_SEG_KERNEL"] = kern
                ms = time_launch(lambda: bs.bs_lookup_ex(idx, dq, m, out, None, reorder=bs.REORDER_SORTED), 2, 5)
                ok = bool(np.array_equal(P.to_numpy_unsigned(out, kb)[samp], want))
                print(json.dumps({"key_bytes": kb, "n": n, "m": m, "m_per_n": m / n, "kernel": kern, "ms": ms,
                                  "G_lookups_per_s": m / ms / 1e6, "ok": ok}), flush=True)
            os.environ.pop("BS_SEG_KERNEL", None)
            idx.close()
            del dk, dq, out
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
