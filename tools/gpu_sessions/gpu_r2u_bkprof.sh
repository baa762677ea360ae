#!/bin/bash
# round 2 (session 2): ncu --set full (source-level) of the BUCKET mode's part / search / unpart / hist kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2u}
mkdir -p $O
CMD="python bench.py --reorder 5 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_bk_(part|search|unpart|hist)" -s 4 -c 4 -o $O/bk $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
