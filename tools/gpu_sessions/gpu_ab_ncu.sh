#!/bin/bash
# per-kernel launch list of two builds (A/B).  usage: gpu_ab_ncu.sh TAG KERNEL_REGEX [bench args]
cd $GRAFT_REPO_ROOT
TAG=$1; K=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
for v in A B; do
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-naive $@"
BS_LIB_PATH=$PWD/paper_2506_01576_b200/lib/libbs_$v.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:$K" -c ${NCU_C:-4} --csv --log-file $O/launches_$v.csv $CMD > $O/ncu_$v.log 2>&1
echo "== $v"; python tools/ncu_kernels.py $O/launches_$v.csv --per 134217728
done
