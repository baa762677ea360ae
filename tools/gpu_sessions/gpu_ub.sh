#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_shfl tools/ubench_shfl.cu
timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,smsp__inst_executed.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum --csv --log-file gpurun_out/ubench_shfl.csv /tmp/ubench_shfl > gpurun_out/ubench_shfl.log 2>&1; echo "rc=$?"
