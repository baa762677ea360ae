#!/bin/bash
# round 2 (session 2): BS_REORDER_BUCKET first run — parity, bench line, per-kernel launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bucket.py -x -q > $O/pytest_bucket.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_bucket.log
timeout 300 python bench.py --reorder 5 --no-e2e --no-naive > $O/bench_bucket.json 2> $O/bench_bucket.err; echo "bench rc=$?"
tail -c 400 $O/bench_bucket.json
CMD="python bench.py --reorder 5 --steps 3 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_bk_ --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1; echo "launch rc=$?"
