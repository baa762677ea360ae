#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_seg.py -x -q > $O/pytest_seg.log 2>&1; echo "seg rc=$?"
timeout 600 python bench.py --config config3 --reorder 4 --steps 20 --no-e2e --no-naive > $O/bench_config3_global.json 2> $O/bench_config3_global.err; echo "c3g rc=$?"
timeout 600 python bench.py --config config3 --steps 20 --no-e2e --no-naive > $O/bench_config3.json 2> $O/bench_config3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config config2 --reorder 4 --steps 20 --no-e2e --no-naive > $O/bench_config2_global.json 2> $O/bench_config2_global.err; echo "c2g rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 6 -c 6 --csv --log-file $O/launches_global.csv python bench.py --config config3 --reorder 4 --steps 2 --warmup 3 --no-e2e --no-naive > $O/ncu_global.log 2>&1; echo "ncu rc=$?"
