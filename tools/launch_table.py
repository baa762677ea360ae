"""Summarise an `ncu --metrics ... --csv` launch list: one line per launch with
time and DRAM / L2-write bytes per query (m = --m)."""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--m", type=float, default=2 ** 27)
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if r and not r[0].startswith("==")]
h = rows[0]
cur = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    k = (int(d["ID"]), d["Kernel Name"].split("(")[0][:48])
    cur.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for k, v in sorted(cur.items()):
    t = v.get("gpu__time_duration.sum", 0) / 1e6
    rd, wr = v.get("dram__bytes_read.sum", 0), v.get("dram__bytes_write.sum", 0)
    print(f"{k[0]:3d} {k[1]:48s} {t:8.3f} ms  DRAM rd {rd / a.m:6.1f} wr {wr / a.m:6.1f} B/q  {(rd + wr) / max(t, 1e-9) / 1e9:7.1f} GB/s")
