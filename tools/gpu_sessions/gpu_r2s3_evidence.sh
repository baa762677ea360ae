#!/bin/bash
# round 2 session 3 evidence: GPU tests, smoke, every bench line (default = BUCKET for config 3),
# per-config DRAM traffic, launch list and ncu --set full of the dominant kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2s3a}
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
B() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "$name rc=$?"; }
B config3_kary --reorder 0 --no-e2e
B config3_sorted --order sorted --no-e2e --no-naive
B config3_global --reorder 4 --no-e2e --no-naive
B config2_sorted --config config2 --order sorted --no-e2e --no-naive
B config2 --config config2
B config1 --config config1 --no-e2e
B config4 --config config4 --steps 5
B config4_kary --config config4 --reorder 0 --steps 3 --no-e2e --no-naive
B config5 --config config5 --steps 5
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum"
K='regex:k_kary_g1|k_seg_sorted|k_peer|k_part|k_seg_part|k_unpart|k_bk_'
run() {  # name, args
  local name=$1; shift
  python bench.py "$@" > $O/plain_$name.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 40 --csv --log-file $O/traffic_$name.csv python bench.py "$@" > $O/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
run c3bucket --steps 1 --warmup 3 --no-e2e --no-naive
run c4bucket --config config4 --steps 1 --warmup 3 --no-e2e --no-naive
run c5bucket --config config5 --steps 1 --warmup 3 --no-e2e --no-dist
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain_launch.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1; echo "launch rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain_full.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_bk_search" -s 3 -c 1 -o $O/bench_kernel $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
