#!/bin/bash
# BUCKET mode iteration: parity tests, bench line, per-kernel launch list.  usage: gpu_bk_iter.sh TAG [extra bench args]
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bucket.py -x -q > $O/pytest_bucket.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_bucket.log
timeout 300 python bench.py --reorder 5 --no-e2e --no-naive "$@" > $O/bench_bucket.json 2> $O/bench_bucket.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/bench_bucket.json').read().strip().splitlines()[-1]);print('G/s',d['value']/1e9,'ms',d['ms_per_step'],'parity',d['parity_sample_ok'],d['invariant_all_ok'])"
CMD="python bench.py --reorder 5 --steps 3 --warmup 3 --no-e2e --no-naive $@"
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_bk_ --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1; echo "launch rc=$?"
python tools/ncu_kernels.py $O/launches.csv --per 134217728
