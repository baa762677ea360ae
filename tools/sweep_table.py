"""Markdown table from tools/size_sweep.py output.

python tools/sweep_table.py profiles/X_size_u32.jsonl profiles/X_size_u64.jsonl
"""
from __future__ import annotations

import json
import sys


def table(path: str) -> str:
    rows = [json.loads(line) for line in open(path) if line.strip()]
    byn: dict[int, dict[str, dict]] = {}
    for r in rows:
        byn.setdefault(r["log2n"], {})[r["variant"]] = r
    kb = rows[0]["key_bytes"]
    out = [f"**u{8 * kb} keys** (G lookups/s, 2^27 random hit queries; build ms = sorted / unsorted input; "
           "footprint = index bytes / array bytes)", "",
           "| log2 n | naive | OPT | K-ary (auto C, mode) | K-ary / naive | build OPT ms | build K-ary ms | footprint K-ary |",
           "|---|---|---|---|---|---|---|---|"]
    for lg, d in sorted(byn.items()):
        nv, op, ka = (d[v]["G_lookups_per_s"] for v in ("naive", "opt", "kary"))
        k = d["kary"]
        ok = all(v["ok"] for v in d.values())
        out.append(f"| {lg} | {nv:.1f} | {op:.1f} | {ka:.1f} (C={k.get('leaf_chunk', '?')}, m{k.get('kary_mode', '?')})"
                   f"{'' if ok else ' PARITY FAIL'} | {ka / nv:.1f}x | "
                   f"{d['opt']['build_ms_sorted_input']:.1f} / {d['opt']['build_ms_unsorted_input']:.1f} | "
                   f"{k['build_ms_sorted_input']:.1f} / {k['build_ms_unsorted_input']:.1f} | "
                   f"{k['footprint_bytes'] / k['array_bytes']:.3f} |")
    return "\n".join(out)


if __name__ == "__main__":
    print("\n\n".join(table(p) for p in sys.argv[1:]))
