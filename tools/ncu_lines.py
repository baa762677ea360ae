"""Aggregate an ncu source page (cuda,sass) by CUDA source line: instructions
executed and stall samples.  python tools/ncu_lines.py rep.ncu-rep [top] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilter = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", *kfilter],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = {}
fname = ""
hdr = None
cur = None
tot_i = tot_s = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1][:90])
        continue
    # sass row under cur
    try:
        samples = int(r[4]); inst = int(r[7])
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += inst
    a[1] += samples
    tot_i += inst
    tot_s += samples
print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{i / tot_i * 100:5.1f}% inst {s / max(tot_s, 1) * 100:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
