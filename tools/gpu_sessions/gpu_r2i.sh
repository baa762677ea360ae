#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2i
mkdir -p $O
CMD="python bench.py --config config3 --reorder 4 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_part<|k_seg_part|k_unpart" -s 3 -c 3 -o $O/global $CMD > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
