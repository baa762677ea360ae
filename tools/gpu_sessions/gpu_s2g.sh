#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x --timeout 600 -k "kary or config1 or edge" > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_parity.log
timeout 900 python tools/sweep.py --what kary --quick --modes 2,3 --kc 9/8,9/16,8/16,5/8,17/16,16/16 --hints 3 --tr 1024/2,1024/4 > gpurun_out/sweep_ti5.jsonl 2> gpurun_out/sweep_ti5.err; echo "sweep rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_ltcfabric.sum,launch__registers_per_thread,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.avg.per_cycle_elapsed
PTS=9/8/2/1024/4,9/16/2/1024/4,9/8/3/1024/4,9/16/3/1024/4,16/16/3/1024/4
timeout 900 ncu --metrics $M --clock-control none -k regex:k_kary --csv --log-file gpurun_out/points4.csv python tools/points.py --pts $PTS > gpurun_out/points4.log 2>&1; echo "ncu points rc=$?"
