#!/bin/bash
# 4-byte peer tags + vectorised finish copy: peer/dist GPU tests, routing paths at config 3 and config-5 per-GPU sizes
set -u
mkdir -p gpurun_out
T=${TAG:-r1s4b}
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_dist.py -q -rf -x --timeout 600 > gpurun_out/${T}_pytest_peer.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest_peer.log
timeout 600 python tools/peer_bench.py > gpurun_out/${T}_peer_bench.jsonl 2>/dev/null; echo "peer rc=$?"; cat gpurun_out/${T}_peer_bench.jsonl
timeout 900 python tools/peer_bench.py --n-log2 30 --m-log2 28 --reps 5 > gpurun_out/${T}_peer_config5_per_gpu.jsonl 2>/dev/null; echo "peer c5 rc=$?"; cat gpurun_out/${T}_peer_config5_per_gpu.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/${T}_peer_launches.csv python tools/peer_bench.py --reps 2 > gpurun_out/${T}_peer_under_ncu.log 2>&1; echo "ncu rc=$?"
