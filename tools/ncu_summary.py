"""Summarise ncu reports (read here, no GPU): key DRAM / L2 / L1 / stall metrics.

python tools/ncu_summary.py gpurun_out/kary_full.ncu-rep [...] [--json out.json] [--lookups N]
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "selected", "not_selected", "math_pipe_throttle",
          "lg_throttle", "mio_throttle", "barrier", "branch_resolving", "dispatch_stall", "no_instructions",
          "tex_throttle", "membar", "drain"]

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def summarize(path: str, lookups: int | None = None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    f = float(v)
                except ValueError:
                    d[k] = v
                    continue
                u = units[i]
                if u in SCALE:
                    f *= SCALE[u]
                    k = k + " [B]"
                elif u == "ms":
                    k = k + " [ms]"
                elif u == "us":
                    f /= 1e3
                    k = k + " [ms]"
                elif u == "ns":
                    f /= 1e6
                    k = k + " [ms]"
                d[k] = f
        st = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in hdr:
                try:
                    st[s] = float(vals[hdr.index(k)].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        d["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.01}
        rd = d.get("dram__bytes_read.sum [B]", 0.0)
        wr = d.get("dram__bytes_write.sum [B]", 0.0)
        d["dram_bytes_per_launch"] = rd + wr
        if lookups:
            d["dram_bytes_per_lookup"] = (rd + wr) / lookups
            lts = d.get("lts__t_sectors_srcunit_tex_op_read.sum")
            if isinstance(lts, float):
                d["l2_sectors_per_lookup"] = lts / lookups
        ms = d.get("gpu__time_duration.sum [ms]")
        if ms:
            d["dram_GBps"] = (rd + wr) / (ms / 1e3) / 1e9
            if lookups:
                d["G_lookups_per_s_under_ncu"] = lookups / (ms / 1e3) / 1e9
        out.append(d)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:]]
    js = None
    lookups = None
    if "--json" in args:
        i = args.index("--json")
        js = args[i + 1]
        del args[i:i + 2]
    if "--lookups" in args:
        i = args.index("--lookups")
        lookups = int(args[i + 1])
        del args[i:i + 2]
    res = {p: summarize(p, lookups) for p in args}
    txt = json.dumps(res, indent=1)
    print(txt)
    if js:
        open(js, "w").write(txt)
