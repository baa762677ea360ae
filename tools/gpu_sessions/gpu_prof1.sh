#!/bin/bash
# ncu --set full of one BUCKET-mode kernel.  usage: gpu_prof1.sh TAG KERNEL_REGEX [bench args]
cd $GRAFT_REPO_ROOT
TAG=$1; K=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-naive $@"
$CMD > $O/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s 3 -c 1 -o $O/prof $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
