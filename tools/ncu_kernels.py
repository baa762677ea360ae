"""Per-kernel summary of an `ncu --metrics ... --csv` launch list: mean of each
metric over the launches of each kernel (optionally per query: --per N)."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = [l for l in open(path) if not l.startswith("==")]
    by = defaultdict(lambda: defaultdict(list))
    order = []
    for r in csv.DictReader(rows):
        k = r["Kernel Name"].split("(")[0]
        if k not in by:
            order.append(k)
        by[k][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
    return order, by


def main():
    path = sys.argv[1]
    per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 0.0
    order, by = load(path)
    for k in order:
        ms = by[k]
        parts = [f"{k[:60]:60s} x{len(next(iter(ms.values())))}"]
        for name, v in ms.items():
            avg = sum(v) / len(v)
            if name == "gpu__time_duration.sum":
                parts.append(f"t={avg / 1e6:.3f}ms" if avg > 1e5 else f"t={avg / 1e3:.1f}us")
            elif per and ("bytes" in name or "sectors" in name or "inst" in name):
                parts.append(f"{name.split('.')[0].split('__')[-1]}={avg / per:.2f}/q")
            else:
                parts.append(f"{name.split('.')[0].split('__')[-1]}={avg:.1f}")
        print("  ".join(parts))


if __name__ == "__main__":
    main()
