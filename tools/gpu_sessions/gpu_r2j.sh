#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2j
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_seg.py -x -q -k global > $O/pytest_seg.log 2>&1; echo "seg rc=$?"
timeout 600 python bench.py --config config3 --reorder 4 --steps 20 --no-e2e --no-naive > $O/bench_config3_global.json 2> $O/bench_config3_global.err; echo "c3g rc=$?"
timeout 600 python bench.py --config config2 --reorder 4 --steps 20 --no-e2e --no-naive > $O/bench_config2_global.json 2> $O/bench_config2_global.err; echo "c2g rc=$?"
CMD="python bench.py --config config3 --reorder 4 --steps 2 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum --clock-control none -k regex:"k_part|k_seg_part|k_unpart" -c 8 --csv --log-file $O/launches_global.csv $CMD > $O/ncu_global.log 2>&1; echo "ncu rc=$?"
