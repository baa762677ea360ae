#!/bin/bash
# round 2 (session 2): random 32-B read cost per PTX load flavour (tools/ubench_flavors.cu), plus a bench sanity line
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2s
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python bench.py --no-e2e > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
./tools/ubench_flavors > $O/flavors.jsonl 2>&1; echo "flavors rc=$?"
./tools/ubench_flavors -1 32 > $O/flavors_fetch32.jsonl 2>&1; echo "flavors32 rc=$?"
M=dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for r in $(seq 0 15); do
  timeout 120 ncu --metrics $M --clock-control none -k regex:gather -s 1 -c 1 --csv --log-file $O/ncu_$r.csv ./tools/ubench_flavors $r > /dev/null 2>&1
done
for r in 8 10 13; do
  timeout 120 ncu --metrics $M --clock-control none -k regex:gather -s 1 -c 1 --csv --log-file $O/ncu_${r}_f32.csv ./tools/ubench_flavors $r 32 > /dev/null 2>&1
done
echo done
