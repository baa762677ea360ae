"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (read
here, no GPU): per-kernel launch count, total/mean ns and share of the run.

python tools/launch_summary.py gpurun_out/X_launches.csv "<the ncu command>" > profiles/X_launches.json
"""
from __future__ import annotations

import csv
import io
import json
import sys
from collections import OrderedDict


def main() -> None:
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = OrderedDict()
    launches = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        name = r["Kernel Name"].split("(")[0]
        d = per.setdefault(name, {"launches": 0, "total_ns": 0.0})
        d["launches"] += 1
        d["total_ns"] += ns
        launches.append({"id": int(r["ID"]), "kernel": name, "grid": r["Grid Size"], "block": r["Block Size"], "ns": ns})
    tot = sum(d["total_ns"] for d in per.values()) or 1.0
    for d in per.values():
        d["mean_ns"] = d["total_ns"] / d["launches"]
        d["share_pct"] = round(100.0 * d["total_ns"] / tot, 2)
    print(json.dumps({"cmd": cmd, "note": "cold-cache serialised launches under ncu; compare shares, not absolutes",
                      "kernels": per, "launches": launches}, indent=1))


if __name__ == "__main__":
    main()
