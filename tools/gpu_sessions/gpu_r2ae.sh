#!/bin/bash
# coarse BUCKET mode: parity, config 4 and config 3 (forced coarse) bench lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2ae}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_bucket.py -x -q > $O/pytest_bucket.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_bucket.log
timeout 600 python bench.py --config config4 --reorder 5 --steps 3 --no-e2e --no-naive > $O/bench_c4_bucket.json 2> $O/bench_c4_bucket.err; echo "c4 rc=$?"
python -c "import json;d=json.loads(open('$O/bench_c4_bucket.json').read().strip().splitlines()[-1]);print('c4 G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
BS_BUCKET_COARSE=1 timeout 300 python bench.py --reorder 5 --no-e2e --no-naive > $O/bench_c3_coarse.json 2> $O/bench_c3_coarse.err; echo "c3c rc=$?"
python -c "import json;d=json.loads(open('$O/bench_c3_coarse.json').read().strip().splitlines()[-1]);print('c3 coarse G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
timeout 300 python bench.py --reorder 5 --no-e2e --no-naive > $O/bench_c3_fine.json 2> $O/bench_c3_fine.err; echo "c3 rc=$?"
python -c "import json;d=json.loads(open('$O/bench_c3_fine.json').read().strip().splitlines()[-1]);print('c3 fine G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
CMD="python bench.py --config config4 --reorder 5 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bk_|k_kary" -c 12 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu.log 2>&1; echo "launch rc=$?"
python tools/ncu_kernels.py $O/launches_c4.csv --per 1073741824
