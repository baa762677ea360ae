#!/bin/bash
# smoke (with peer + merge), peer-path launch list under ncu
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3j_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s3j_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_peer|k_kary_g1|k_route|k_unroute|k_add|nccl" -c 60 --csv --log-file gpurun_out/s3j_peer_launches.csv python tools/peer_bench.py --reps 2 > gpurun_out/s3j_peer_under_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/s3j_peer_under_ncu.log
