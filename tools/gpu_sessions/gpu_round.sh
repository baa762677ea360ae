#!/bin/bash
# Round checkpoint on one B200: tests, smoke, bench lines, launch list, ncu of the bench kernel.
set -u
mkdir -p gpurun_out
T=${TAG:-r1}
timeout 1200 python -m pytest tests -m gpu -q -rf -x --timeout 900 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cat gpurun_out/${T}_bench.json
timeout 900 python bench.py --order sorted --no-e2e > gpurun_out/${T}_bench_sorted.json 2> gpurun_out/${T}_bench_sorted.err; echo "bench sorted rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "bench ref rc=$?"; cat gpurun_out/${T}_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e > gpurun_out/${T}_bench_under_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_kary -s 2 -c 1 -o gpurun_out/${T}_bench_kernel -f \
    python tools/one_launch.py --variant kary --k 5 --c 16 --mode 7 --threads 1024 --nreg 4 --hints 7 > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
