#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x --timeout 600 -k "opt or host or config1 or edge" > gpurun_out/pytest_l.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_l.log
timeout 900 python tools/e2e_sweep.py > gpurun_out/e2e_sweep.jsonl 2> gpurun_out/e2e_sweep.err; echo "e2e rc=$?"
timeout 900 python tools/sweep.py --config config2 --what ladder > gpurun_out/ladder_c2_l1b.jsonl 2> gpurun_out/ladder_c2_l1b.err; echo "ladder rc=$?"
timeout 900 python tools/sweep.py --config config3 --what ladder > gpurun_out/ladder_c3_l1b.jsonl 2> gpurun_out/ladder_c3_l1b.err; echo "ladder rc=$?"
