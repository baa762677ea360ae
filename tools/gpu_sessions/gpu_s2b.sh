#!/bin/bash
# Tiered K-ary: parity + sweep + ncu of the best point.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x --timeout 600 -k "kary" > gpurun_out/pytest_kary.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_kary.log
timeout 1200 python tools/sweep.py --what kary --quick --modes 2 --kc 17/16,16/16,9/16,5/8,9/8,33/32,16/32,8/16 --hints 3 --tr 1024/1,1024/2,1024/4,512/2,512/4 > gpurun_out/sweep_ti.jsonl 2> gpurun_out/sweep_ti.err; echo "sweep rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/kary_ti_K17C16 -f \
    python tools/one_launch.py --variant kary --k 17 --c 16 --mode 2 --threads 1024 --nreg 2 > gpurun_out/ncu_ti.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/kary_ti_K5C8 -f \
    python tools/one_launch.py --variant kary --k 5 --c 8 --mode 2 --threads 1024 --nreg 2 > gpurun_out/ncu_ti2.log 2>&1; echo "ncu full rc=$?"
