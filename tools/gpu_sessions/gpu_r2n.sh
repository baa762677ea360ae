#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2n
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_seg.py -x -q -k global > $O/pytest_seg.log 2>&1; echo "seg rc=$?"
timeout 600 python bench.py --config config3 --reorder 4 --steps 20 --no-e2e --no-naive > $O/bench_config3_global.json 2> $O/bench_config3_global.err; echo "c3g rc=$?"
CMD="python bench.py --config config3 --reorder 4 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain_full.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_part$|^k_unpart$" -s 2 -c 2 -o $O/kpart $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
