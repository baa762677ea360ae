#!/bin/bash
# GPU probe: random-gather microbenchmark, knob sweep, ncu captures (run under gpurun).
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_gather tools/ubench_gather.cu && \
  timeout 300 /tmp/ubench_gather > gpurun_out/ubench_gather.jsonl 2>&1
echo "ubench rc=$?"
timeout 900 python tools/sweep.py --what naive,kary,opt --quick > gpurun_out/sweep_quick.jsonl 2> gpurun_out/sweep_quick.err
echo "sweep rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/kary_full -f \
  python tools/one_launch.py --variant kary > gpurun_out/ncu_kary.log 2>&1
echo "ncu kary rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_naive -s 2 -c 1 -o gpurun_out/naive_full -f \
  python tools/one_launch.py --variant naive > gpurun_out/ncu_naive.log 2>&1
echo "ncu naive rc=$?"
