#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -rf -x --timeout 600 > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_k.log
timeout 900 python tools/sweep.py --what kary --quick --modes 7 --kc 5/16,4/16,9/16 --hints 3 --tr 1024/4,1024/52 > gpurun_out/sweep_g1p.jsonl 2> gpurun_out/sweep_g1p.err; echo "sweep rc=$?"
timeout 900 python tools/sweep.py --config config3 --what ladder > gpurun_out/ladder_c3_l1.jsonl 2> gpurun_out/ladder_c3_l1.err; echo "ladder rc=$?"
timeout 900 python tools/sweep.py --config config2 --what ladder > gpurun_out/ladder_c2_l1.jsonl 2> gpurun_out/ladder_c2_l1.err; echo "ladder rc=$?"
