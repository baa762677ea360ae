#!/bin/bash
# leaf chunk vs size: one 32-B sector / 64 B / one 128-B line, modes 6 and 7
set -u
mkdir -p gpurun_out
timeout 1500 python tools/mode_sweep.py --kb 4 --lo 18 --hi 28 --step 2 --modes 6,7 --kc 5/8,5/16,5/32 > gpurun_out/s3x_kc_u32.jsonl 2> gpurun_out/s3x.err; echo "u32 rc=$?"
timeout 1500 python tools/mode_sweep.py --kb 8 --lo 18 --hi 26 --step 2 --modes 6,7 --kc 5/4,5/8,5/16 > gpurun_out/s3x_kc_u64.jsonl 2>> gpurun_out/s3x.err; echo "u64 rc=$?"; tail -2 gpurun_out/s3x.err
