#!/bin/bash
# round 2, call b: GPU tests after the boundary changes + the new bench in every config (N=1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in config3 config2 config1; do
  timeout 600 python bench.py --config $c --steps 20 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --config config3 --order sorted --steps 20 --no-e2e > $O/bench_config3_sorted.json 2> $O/bench_config3_sorted.err; echo "sorted rc=$?"
timeout 900 python bench.py --config config4 --steps 5 > $O/bench_config4.json 2> $O/bench_config4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config config5 --steps 5 > $O/bench_config5.json 2> $O/bench_config5.err; echo "c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
