#!/bin/bash
set -u
mkdir -p gpurun_out
for cfg in "16 16 3 4" "16 16 2 4"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/ti_K$1_C$2_m$3 -f \
    python tools/one_launch.py --variant kary --k $1 --c $2 --mode $3 --threads 1024 --nreg $4 > gpurun_out/ncu_ti.log 2>&1; echo "ncu $cfg rc=$?"
done
