#!/bin/bash
# leaf chunk 8 vs 16 (u64): sustained bench (power) + DRAM bytes per lookup
set -u
mkdir -p gpurun_out
for C in 16 8; do
  timeout 600 python bench.py --no-e2e --no-naive --leaf-chunk $C --steps 200 > gpurun_out/s3h_bench_C$C.json 2> gpurun_out/s3h_bench_C$C.err; echo "bench C=$C rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/s3h_bench_C$C.json'));print($C, round(d['value']/1e9,2), d['clocks'])"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_kary -s 2 -c 1 --csv python tools/one_launch.py --variant kary --k 5 --c $C --mode 6 --threads 1024 --nreg 4 --hints 7 > gpurun_out/s3h_ncu_C$C.csv 2>&1; echo "ncu rc=$?"; grep -E "dram__bytes|duration|hit_rate" gpurun_out/s3h_ncu_C$C.csv | cut -d, -f13-16
done
