#!/bin/bash
# round-end evidence: checkpoint (tests, smoke, bench lines, launch list, ncu), config 2, size sweeps, routing paths
set -u
T=${TAG:-r1final}
TAG=$T bash tools/gpu_sessions/gpu_round.sh
timeout 600 python bench.py --config config2 --no-e2e > gpurun_out/${T}_bench_config2.json 2>/dev/null; echo "c2 rc=$?"
timeout 600 python tools/peer_bench.py > gpurun_out/${T}_peer_bench.jsonl 2>/dev/null; echo "peer rc=$?"
timeout 1500 python tools/size_sweep.py --kb 4 --lo 15 --hi 29 --step 1 > gpurun_out/${T}_size_u32.jsonl 2>/dev/null; echo "u32 rc=$?"
timeout 1500 python tools/size_sweep.py --kb 8 --lo 16 --hi 30 --step 1 > gpurun_out/${T}_size_u64.jsonl 2>/dev/null; echo "u64 rc=$?"
