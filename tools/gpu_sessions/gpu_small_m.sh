#!/bin/bash
# BUCKET at the strong-scaling per-rank batch (2^24, N = 8): per-kernel launch list vs the event-timed call.
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python tools/bucket_sweep.py --kb 8 --lo 26 --hi 26 --m-log2 24 > $O/sweep24.jsonl 2> $O/sweep24.err; cat $O/sweep24.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bk_" --csv --log-file $O/launches24.csv python tools/bucket_sweep.py --kb 8 --lo 26 --hi 26 --m-log2 24 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_kernels.py $O/launches24.csv --per 16777216
