#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/ti_K16_C16_m2b -f \
    python tools/one_launch.py --variant kary --k 16 --c 16 --mode 2 --threads 1024 --nreg 4 > gpurun_out/ncu_ti.log 2>&1; echo "ncu rc=$?"
