"""Read an ncu --csv metrics log of tools/points.py (2 launches per point) -> JSON lines.

python tools/ncu_points.py gpurun_out/points.csv gpurun_out/points.log [--m 134217728]
"""
from __future__ import annotations

import csv
import collections
import json
import sys


def main():
    csvp, logp = sys.argv[1], sys.argv[2]
    m = int(sys.argv[sys.argv.index("--m") + 1]) if "--m" in sys.argv else 1 << 27
    rows = list(csv.reader(open(csvp)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        k = int(d["ID"])
        per.setdefault(k, {"kernel": d["Kernel Name"]})
        v = d["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            pass
        per[k][d["Metric Name"] + (f" [{d['Metric Unit']}]" if d["Metric Unit"] else "")] = v
    pts = [json.loads(l) for l in open(logp) if l.startswith("{")]
    launches = [v for v in per.values() if "k_kary" in v["kernel"]]
    for i, pt in enumerate(pts):
        if 2 * i + 1 >= len(launches):
            break
        L = launches[2 * i + 1]
        rec = dict(pt)
        rec["kernel"] = L["kernel"].split("(")[0]
        for k, v in L.items():
            if k == "kernel":
                continue
            rec[k] = v
        t = [v for k, v in L.items() if k.startswith("gpu__time_duration.sum")][0]
        unit = [k for k in L if k.startswith("gpu__time_duration.sum")][0]
        ns = t * (1e6 if "msecond" in unit else 1e3 if "usecond" in unit else 1.0)
        dr = sum(v * (1e9 if "Gbyte" in k else 1e6 if "Mbyte" in k else 1e3 if "Kbyte" in k else 1)
                 for k, v in L.items() if k.startswith("dram__bytes_"))
        rec["G_lookups_per_s_under_ncu"] = m / ns
        rec["dram_B_per_lookup"] = dr / m
        rec["dram_GBps"] = dr / ns
        inst = [v for k, v in L.items() if k.startswith("smsp__inst_executed.sum")]
        if inst:
            rec["inst_per_lookup"] = inst[0] / m
        print(json.dumps(rec))


if __name__ == "__main__":
    main()
