#!/bin/bash
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_gather tools/ubench_gather.cu
timeout 300 /tmp/ubench_gather > gpurun_out/ubench3.jsonl 2>&1; echo "ubench rc=$?"
M=dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ubench3_ncu.csv /tmp/ubench_gather > /dev/null 2>&1; echo "ncu ubench rc=$?"
timeout 1200 python tools/sweep.py --what naive,kary,opt --quick --kc 5/8,9/8,17/16,5/4,3/4,9/16,17/8 --hints 3,7 > gpurun_out/sweep3.jsonl 2> gpurun_out/sweep3.err
echo "sweep rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/kary3_K5_C8 -f \
    python tools/one_launch.py --variant kary --k 5 --c 8 --threads 512 --nreg 8 --hints 7 > /dev/null 2>&1; echo "ncu rc=$?"
