#!/bin/bash
# tie-fix check: K-ary parity tests, bench (no regression), size sweep u64 + u32 with build times
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -rf -x --timeout 600 > gpurun_out/s3e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3e_pytest.log
timeout 600 python bench.py --no-e2e --steps 50 > gpurun_out/s3e_bench.json 2> gpurun_out/s3e_bench.err; echo "bench rc=$?"; cut -c1-330 gpurun_out/s3e_bench.json
timeout 1500 python tools/size_sweep.py --kb 8 --lo 16 --hi 30 --step 2 > gpurun_out/s3e_size_u64.jsonl 2> gpurun_out/s3e_size_u64.err; echo "u64 rc=$?"; tail -3 gpurun_out/s3e_size_u64.err
timeout 1500 python tools/size_sweep.py --kb 4 --lo 15 --hi 29 --step 2 > gpurun_out/s3e_size_u32.jsonl 2> gpurun_out/s3e_size_u32.err; echo "u32 rc=$?"; tail -3 gpurun_out/s3e_size_u32.err
