#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "narrow or config1 or edge or kary" > $O/pytest_parity.log 2>&1; echo "par rc=$?"
timeout 600 python tools/tie_bench.py > $O/tie_bench.jsonl 2> $O/tie_bench.err; echo "tie rc=$?"
timeout 600 python bench.py --config config3 --steps 20 --no-e2e > $O/bench_config3.json 2> $O/bench_config3.err; echo "c3 rc=$?"
