#!/bin/bash
# round 2, call a: random-gather microbenchmark (granularity / lane layout) + DRAM bytes per access
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
./tools/ubench_gather2 > $O/ubench.jsonl 2>&1
for k in 0 1 2 3 4 5 6 9 10 11 12 13 14 15; do
  ./tools/ubench_gather2 $k > $O/plain_$k.log 2>&1 && \
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --clock-control none -k regex:gather -s 1 -c 1 --csv --log-file $O/ncu_$k.csv ./tools/ubench_gather2 $k > /dev/null 2>&1
done
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
echo done
