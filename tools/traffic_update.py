"""Fold `ncu --metrics` launch lists of bench.py runs (tools/gpu_r2k.sh:
gpurun_out/<tag>/traffic_<name>.csv) into profiles/traffic.json, keyed like
bench.py's roofline.traffic_key.  Per step: the LAST launch of each kernel
name (after bench.py's warm-up steps), summed over the step's kernels.

python tools/traffic_update.py gpurun_out/r2k
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {   # run name -> (traffic key, queries per launch, kernels of one step)
    "c3": ("config3/random/kary/K5/C16/mode7", 1 << 27, ["k_kary_g1"]),
    "c3sorted": ("config3/sorted/kary/K5/C16/mode7/r3", 1 << 27, ["k_seg_sorted"]),
    "c2": ("config2/random/kary/K5/C8/mode7", 1 << 27, ["k_kary_g1"]),
    "c4": ("config4/random/kary/K5/C16/mode7", 1 << 30, ["k_kary_g1"]),
    "c5": ("config5/random/kary/K5/C16/mode7/peer", 1 << 28, ["k_peer_route", "k_kary_g1", "k_peer_finish"]),
    "c3global": ("config3/random/kary/K5/C16/mode7/r4", 1 << 27, ["k_part", "k_seg_part", "k_part_ovf", "k_unpart"]),
    "c3bucket": ("config3/random/kary/K5/C16/mode7/r5", 1 << 27,
                 ["k_bk_hist", "k_bk_scan", "k_bk_part", "k_bk_search", "k_bk_unpart"]),
    "c4bucket": ("config4/random/kary/K5/C16/mode7/r5", 1 << 30,
                 ["k_bk_hist", "k_bk_scan", "k_bk_part", "k_bk_search", "k_bk_unpart"]),
    "c5bucket": ("config5/random/kary/K5/C16/mode7/peer/r5", 1 << 28,
                 ["k_peer_route", "k_peer_wait", "k_bk_hist", "k_bk_scan", "k_bk_part", "k_bk_search", "k_bk_unpart",
                  "k_peer_finish"]),
}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = int(d["ID"])
        out.setdefault(k, {"kernel": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [out[k] for k in sorted(out)]


def main(tag_dir):
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    for name, (key, m, kernels) in KEYS.items():
        p = os.path.join(tag_dir, f"traffic_{name}.csv")
        if not os.path.exists(p):
            continue
        L = launches(p)
        step = []
        for kn in kernels:
            mine = [x for x in L if x["kernel"].startswith("void " + kn + "<") or x["kernel"].startswith(kn + "(")
                    or x["kernel"].startswith("void " + kn + "(")]
            if mine:
                step.append(mine[-1])
        if not step:
            continue
        dram = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in step)
        t = sum(x["gpu__time_duration.sum"] for x in step) / 1e6
        l2s = sum(x.get("lts__t_sectors_srcunit_tex_op_read.sum", 0) for x in step)
        tj[key] = {
            "dram_bytes_per_launch": dram, "queries": m, "dram_bytes_per_lookup": dram / m,
            "l2_read_sectors_per_lookup": l2s / m, "ncu_ms": t,
            "kernels": [{"kernel": x["kernel"].split("(")[0], "ms": x["gpu__time_duration.sum"] / 1e6,
                         "dram_B_per_lookup": (x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"]) / m,
                         "lts_pct": x.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                         "l1tex_pct": x.get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                         "l2_hit_pct": x.get("lts__t_sector_hit_rate.pct")} for x in step],
            "source": f"{os.path.relpath(p, ROOT)} (ncu --metrics, last launch of each kernel after bench.py's warm-up)",
        }
        print(key, f"{dram / m:.1f} DRAM B/lookup, {t:.3f} ms under ncu")
    json.dump(tj, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
