#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d
mkdir -p $O
timeout 600 python bench.py --config config3 --steps 20 --no-e2e > $O/bench_config3.json 2> $O/bench_config3.err; echo "c3 rc=$?"
timeout 900 python -X faulthandler bench.py --config config5 --steps 5 --verbose > $O/bench_config5.json 2> $O/bench_config5.err; echo "c5 rc=$?"
