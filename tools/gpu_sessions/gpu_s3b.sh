#!/bin/bash
# fused peer routing: parity tests, routing overhead at world 1, bench sanity
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_dist.py -q -rf -x --timeout 600 > gpurun_out/s3b_pytest_peer.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/s3b_pytest_peer.log
timeout 600 python tools/peer_bench.py > gpurun_out/s3b_peer_bench.jsonl 2> gpurun_out/s3b_peer_bench.err; echo "peer bench rc=$?"; cat gpurun_out/s3b_peer_bench.jsonl; tail -5 gpurun_out/s3b_peer_bench.err
timeout 600 python bench.py --no-e2e --steps 50 > gpurun_out/s3b_bench.json 2> gpurun_out/s3b_bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/s3b_bench.json
