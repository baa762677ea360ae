#!/bin/bash
# Session-2 probe: GPU tests, bench line, K-ary hybrid vs warp sweep, L2 fetch granularity, ncu.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --k 5 --leaf-chunk 8 > gpurun_out/bench_k5c8.json 2> gpurun_out/bench_k5c8.err; echo "bench rc=$?"; cat gpurun_out/bench_k5c8.json
timeout 1200 python tools/sweep.py --what kary --quick --modes 1,0 --kc 5/8,9/16,9/8,3/4,17/16 --hints 3 --tr 256/1,256/2,256/4,512/2,512/4,512/8,1024/2,1024/4 > gpurun_out/sweep_hy.jsonl 2> gpurun_out/sweep_hy.err; echo "sweep rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_gather tools/ubench_gather.cu
timeout 300 /tmp/ubench_gather 32 > gpurun_out/ubench_f32.jsonl 2>&1; echo "ubench32 rc=$?"
M=dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ubench_ncu_f32.csv /tmp/ubench_gather 32 > /dev/null 2>&1; echo "ncu ubench32 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --k 5 --leaf-chunk 8 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_under_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/kary_hy_K5C8 -f \
    python tools/one_launch.py --variant kary --k 5 --c 8 > gpurun_out/ncu_hy.log 2>&1; echo "ncu full rc=$?"
