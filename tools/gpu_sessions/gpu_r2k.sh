#!/bin/bash
# round 2, call k: ncu of k_part; per-config DRAM traffic of the timed kernels; build sweep
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2k
mkdir -p $O
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum"
K='regex:k_kary_g1|k_seg_sorted|k_peer|k_part|k_seg_part|k_unpart'
run() {  # name, args
  local name=$1; shift
  python bench.py "$@" > $O/plain_$name.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 40 --csv --log-file $O/traffic_$name.csv python bench.py "$@" > $O/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
run c3 --config config3 --steps 1 --warmup 3 --no-e2e --no-naive
run c3sorted --config config3 --order sorted --reorder 3 --steps 1 --warmup 3 --no-e2e --no-naive
run c2 --config config2 --steps 1 --warmup 3 --no-e2e --no-naive
run c4 --config config4 --steps 1 --warmup 3 --no-e2e --no-naive
run c5 --config config5 --steps 1 --warmup 3 --no-e2e --no-dist
run c3global --config config3 --reorder 4 --steps 1 --warmup 3 --no-e2e --no-naive
CMD="python bench.py --config config3 --reorder 4 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain_full.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_part<" -s 3 -c 1 -o $O/kpart $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
timeout 1500 python tools/build_sweep.py --lo 15 --hi 30 --reps 3 > $O/build_sweep.jsonl 2> $O/build_sweep.err; echo "build rc=$?"
