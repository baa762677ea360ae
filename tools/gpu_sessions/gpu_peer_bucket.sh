#!/bin/bash
# Peer path with the bucket pipeline (config 5): parity tests, config-5 bench
# lines (bucket default vs the K-ary peer kernel), per-kernel launch list.
# usage: gpu_peer_bucket.sh TAG
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > $O/pytest_peer.log 2>&1; echo "pytest peer rc=$?"
tail -3 $O/pytest_peer.log
for R in 5 0; do
  timeout 600 python bench.py --config config5 --reorder $R --no-e2e --no-naive > $O/bench_c5_r$R.json 2> $O/bench_c5_r$R.err; echo "bench r$R rc=$?"
  python -c "import json;d=json.loads(open('$O/bench_c5_r$R.json').read().strip().splitlines()[-1]);print('r$R G/s',d['value']/1e9,'ms',d['ms_per_step'],'parity',d.get('parity_sample_ok'),d.get('invariant_all_ok'),'nccl',d.get('nccl_path',{}).get('value'))"
done
CMD="python bench.py --config config5 --steps 2 --warmup 3 --no-e2e --no-naive --no-dist"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bk_|k_peer" --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1; echo "launch rc=$?"
python tools/ncu_kernels.py $O/launches.csv --per 268435456
