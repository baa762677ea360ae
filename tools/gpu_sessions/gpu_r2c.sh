#!/bin/bash
# round 2, call c: ordered-batch path parity + timing, fullsize tests, carve-out fix
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_seg.py -x -q > $O/pytest_seg.log 2>&1; echo "seg rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > $O/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"
timeout 600 python bench.py --config config3 --steps 20 --no-e2e > $O/bench_config3.json 2> $O/bench_config3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config config3 --order sorted --reorder 3 --steps 20 --no-e2e --no-naive > $O/bench_config3_sorted_seg.json 2> $O/bench_config3_sorted_seg.err; echo "c3s rc=$?"
timeout 600 python bench.py --config config2 --order sorted --reorder 3 --steps 20 --no-e2e --no-naive > $O/bench_config2_sorted_seg.json 2> $O/bench_config2_sorted_seg.err; echo "c2s rc=$?"
timeout 600 python bench.py --config config3 --reorder 3 --steps 5 --no-e2e --no-naive > $O/bench_config3_random_seg.json 2> $O/bench_config3_random_seg.err; echo "c3r rc=$?"
timeout 900 python bench.py --config config5 --steps 5 > $O/bench_config5.json 2> $O/bench_config5.err; echo "c5 rc=$?"
