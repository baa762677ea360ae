#!/bin/bash
# config 2 (2^20 u32, L2-resident): leaf size / fan-out for the thread-per-lookup schedules
set -u
mkdir -p gpurun_out
timeout 1200 python tools/sweep.py --config config2 --order random --what kary --quick --hints 7 --modes 6,7 --kc 5/32,5/16,5/8,9/16,9/8,17/32,4/8,3/8 --tr 1024/4 > gpurun_out/s3w_c2_kc.jsonl 2> gpurun_out/s3w.err; echo "rc=$?"; tail -2 gpurun_out/s3w.err
python - <<'PY'
import json
for l in open("gpurun_out/s3w_c2_kc.jsonl"):
    d = json.loads(l); print(d.get("mode"), d.get("K"), d.get("C"), round(d.get("glookups_per_s", 0), 1), d.get("ok"))
PY
