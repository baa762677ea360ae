#!/bin/bash
# final-session evidence: config-4 bench line, size sweeps at the current schedule defaults
set -u
mkdir -p gpurun_out
T=${TAG:-r1s4e}
timeout 900 python bench.py --config config4 --no-e2e --steps 30 > gpurun_out/${T}_bench_config4.json 2>/dev/null; echo "c4 rc=$?"; cat gpurun_out/${T}_bench_config4.json
timeout 1500 python tools/size_sweep.py --kb 8 --lo 16 --hi 30 --step 1 > gpurun_out/${T}_size_u64.jsonl 2>/dev/null; echo "u64 rc=$?"
timeout 1500 python tools/size_sweep.py --kb 4 --lo 15 --hi 29 --step 1 > gpurun_out/${T}_size_u32.jsonl 2>/dev/null; echo "u32 rc=$?"
