#!/bin/bash
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_gather tools/ubench_gather.cu
timeout 300 /tmp/ubench_gather 32 > gpurun_out/ubench_gather_f32.jsonl 2>&1; echo "ubench32 rc=$?"
M=dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ubench_ncu_default.csv /tmp/ubench_gather > /dev/null 2>&1; echo "ncu ubench rc=$?"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ubench_ncu_f32.csv /tmp/ubench_gather 32 > /dev/null 2>&1; echo "ncu ubench32 rc=$?"
for cfg in "5 8 512 8" "9 8 1024 4" "17 16 1024 4"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/kary_K$1_C$2_t$3_R$4 -f \
    python tools/one_launch.py --variant kary --k $1 --c $2 --threads $3 --nreg $4 > gpurun_out/ncu_kary_K$1.log 2>&1
  echo "ncu kary $cfg rc=$?"
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_kary -s 2 -c 1 --csv --log-file gpurun_out/kary_K$1_C$2_f32.csv \
    python tools/one_launch.py --variant kary --k $1 --c $2 --threads $3 --nreg $4 --l2fetch 32 > /dev/null 2>&1
done
timeout 900 python tools/sweep.py --what kary --quick --kc 3/4,3/8,5/4,5/8,5/16,9/4,9/8,9/16,17/8 > gpurun_out/sweep_kary2.jsonl 2> gpurun_out/sweep_kary2.err
echo "sweep rc=$?"
