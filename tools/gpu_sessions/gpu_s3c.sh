#!/bin/bash
# Figs. 11-13 analogue: lookup throughput, build time and footprint vs build size
set -u
mkdir -p gpurun_out
timeout 1500 python tools/size_sweep.py --kb 4 --lo 15 --hi 29 --step 2 > gpurun_out/s3c_size_u32.jsonl 2> gpurun_out/s3c_size_u32.err; echo "u32 rc=$?"; tail -3 gpurun_out/s3c_size_u32.err
timeout 1500 python tools/size_sweep.py --kb 8 --lo 16 --hi 30 --step 2 > gpurun_out/s3c_size_u64.jsonl 2> gpurun_out/s3c_size_u64.err; echo "u64 rc=$?"; tail -3 gpurun_out/s3c_size_u64.err
wc -l gpurun_out/s3c_size_*.jsonl
