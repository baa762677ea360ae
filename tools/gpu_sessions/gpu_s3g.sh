#!/bin/bash
# g1 MLP: T = 2 lookups per thread at 768 threads (80 regs) vs T = 1 at 1024 / 768 threads
set -u
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --config config3 --order random --what kary --quick --hints 3,7 --modes 6 --kc 5/16 --tr 1024/4,768/4,768/36,768/34,768/33,1024/2 > gpurun_out/s3g_sweep_T2.jsonl 2> gpurun_out/s3g_sweep_T2.err; echo "sweep rc=$?"; tail -3 gpurun_out/s3g_sweep_T2.err
python - <<'PY'
import json
for l in open("gpurun_out/s3g_sweep_T2.jsonl"):
    d = json.loads(l); print(d.get("K"), d.get("C"), d.get("threads"), d.get("R"), d.get("hints"), round(d.get("glookups_per_s", 0), 2), d.get("ok"))
PY
timeout 600 python bench.py --no-e2e --steps 50 > gpurun_out/s3g_bench.json 2> gpurun_out/s3g_bench.err; echo "bench rc=$?"; cut -c1-900 gpurun_out/s3g_bench.json
