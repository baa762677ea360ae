#!/bin/bash
# K-ary vs BUCKET over the array size (u64 and u32), m = 2^27 random hits.  usage: gpu_bucket_sweep.sh TAG
cd $GRAFT_REPO_ROOT
O=gpurun_out/$1
mkdir -p $O
timeout 1500 python tools/bucket_sweep.py --kb 8 --lo 20 --hi 30 > $O/bucket_sweep_u64.jsonl 2> $O/bucket_sweep_u64.err; echo "u64 rc=$?"
timeout 1500 python tools/bucket_sweep.py --kb 4 --lo 20 --hi 30 > $O/bucket_sweep_u32.jsonl 2> $O/bucket_sweep_u32.err; echo "u32 rc=$?"
