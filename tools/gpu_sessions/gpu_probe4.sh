#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -x --timeout 900 > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
timeout 1200 python tools/sweep.py --what kary --quick --modes 1 --kc 5/16,5/8,9/16,9/8,17/16,3/8 --hints 3,7 --tr 512/4,1024/4,1024/2,768/4,512/8,1024/8 > gpurun_out/sweep4.jsonl 2> gpurun_out/sweep4.err
echo "sweep rc=$?"
