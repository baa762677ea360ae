"""Per-kernel registers / spills from `python -m paper_2506_01576_b200.build --ptxas --force` output on stdin."""
import re
import subprocess
import sys

txt = sys.stdin.read()
cur = None
res = {}
for line in txt.splitlines():
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        res.setdefault(cur, {})["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        res.setdefault(cur, {})["regs"] = int(m.group(1))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in sorted(res.items()):
    if pat in k:
        try:
            d = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        except Exception:
            d = k
        print(v.get("regs"), v.get("spill"), d[:150])
