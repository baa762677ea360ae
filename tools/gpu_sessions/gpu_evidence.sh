#!/bin/bash
# §4 ladder + K-ary on config 2 (L2-resident u32) and config 3 (random / pre-sorted)
set -u
mkdir -p gpurun_out
T=${TAG:-ev}
for cfg in "config2 random" "config3 random" "config3 sorted"; do
  set -- $cfg
  timeout 1200 python tools/sweep.py --config $1 --order $2 --what ladder > gpurun_out/${T}_ladder_$1_$2.jsonl 2> gpurun_out/${T}_ladder_$1_$2.err; echo "ladder $cfg rc=$?"
  timeout 1200 python tools/sweep.py --config $1 --order $2 --what kary --quick --modes 6,2,0 --kc 5/16,9/16,16/16,17/16 --tr 1024/4,512/4 > gpurun_out/${T}_kary_$1_$2.jsonl 2> gpurun_out/${T}_kary_$1_$2.err; echo "kary $cfg rc=$?"
done
