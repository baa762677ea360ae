#!/bin/bash
set -u
mkdir -p gpurun_out
for cfg in "9 16" "9 8"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/ti_K$1_C$2 -f \
    python tools/one_launch.py --variant kary --k $1 --c $2 --mode 2 --threads 1024 --nreg 4 > gpurun_out/ncu_ti_K$1_C$2.log 2>&1; echo "ncu $cfg rc=$?"
done
