#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2ar}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_bucket.py -x -q > $O/pytest_bucket.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_bucket.log
for c in config3 config4; do
timeout 600 python bench.py --config $c --steps 5 --no-e2e --no-naive > $O/bench_$c.json 2> $O/bench_$c.err
python -c "import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
done
CMD="python bench.py --config config4 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bk_search" -c 2 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu.log 2>&1; echo "launch rc=$?"
python tools/ncu_kernels.py $O/launches_c4.csv --per 1073741824
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bk_search" -c 2 --csv --log-file $O/launches_c3.csv $CMD > $O/ncu3.log 2>&1; echo "launch rc=$?"
python tools/ncu_kernels.py $O/launches_c3.csv --per 134217728
