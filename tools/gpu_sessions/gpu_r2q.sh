#!/bin/bash
# round 2 evidence checkpoint: full GPU tests, smoke, every bench line, L2 roof microbenchmark, launch list + ncu of the bench kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2q
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
B() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "$name rc=$?"; }
B config3_sorted_seg --order sorted --reorder 3 --no-e2e
B config3_sorted_kary --order sorted --no-e2e --no-naive
B config3_global --reorder 4 --no-e2e --no-naive
B config2 --config config2
B config2_sorted_seg --config config2 --order sorted --reorder 3 --no-e2e --no-naive
B config1 --config config1 --no-e2e
B config4 --config config4 --steps 5
B config5 --config config5 --steps 5
./tools/ubench_gather2 > $O/ubench.jsonl 2>&1
for k in 0 1 3 4; do
  ./tools/ubench_gather2 $k > $O/ub_plain_$k.log 2>&1 && \
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gather -s 1 -c 1 --csv --log-file $O/ub_ncu_$k.csv ./tools/ubench_gather2 $k > /dev/null 2>&1
done
echo "ub done"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain_launch.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1; echo "launch rc=$?"
$CMD > $O/plain_full.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_kary_g1$" -s 3 -c 1 -o $O/bench_kernel $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
