#!/bin/bash
# two-level buckets: parity, config 4 and config 3 (forced two-level) bench lines, config 4 launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2aq}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_bucket.py -x -q > $O/pytest_bucket.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_bucket.log
timeout 600 python bench.py --config config4 --steps 3 --no-e2e --no-naive > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
python -c "import json;d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1]);print('c4 G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
BS_BUCKET_TWO=1 timeout 300 python bench.py --no-e2e --no-naive > $O/bench_c3two.json 2> $O/bench_c3two.err; echo "c3two rc=$?"
python -c "import json;d=json.loads(open('$O/bench_c3two.json').read().strip().splitlines()[-1]);print('c3 two-level G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
CMD="python bench.py --config config4 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bk_" -c 12 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu.log 2>&1; echo "launch rc=$?"
python tools/ncu_kernels.py $O/launches_c4.csv --per 1073741824
