#!/bin/bash
# full-size parity (configs 2/3/4, random + sorted), §8f f3 pre-sort comparator, config-4 bench line
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -rf -x --timeout 1400 > gpurun_out/s3d_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -4 gpurun_out/s3d_fullsize.log
timeout 900 python tools/presort_bench.py > gpurun_out/s3d_presort.jsonl 2> gpurun_out/s3d_presort.err; echo "presort rc=$?"; cat gpurun_out/s3d_presort.jsonl; tail -3 gpurun_out/s3d_presort.err
timeout 900 python bench.py --config config4 --no-e2e --steps 20 > gpurun_out/s3d_bench_config4.json 2> gpurun_out/s3d_bench_config4.err; echo "bench c4 rc=$?"; cut -c1-300 gpurun_out/s3d_bench_config4.json; tail -3 gpurun_out/s3d_bench_config4.err
