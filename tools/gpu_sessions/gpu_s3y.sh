#!/bin/bash
# auto leaf chunk: full GPU suite, bench lines on configs 3 and 2, size sweep with the new defaults
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 900 > gpurun_out/s3y_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s3y_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3y_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s3y_smoke.log
timeout 600 python bench.py --no-e2e > gpurun_out/s3y_bench.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s3y_bench.json'));print('c3', round(d['value']/1e9,2), d['config']['leaf_chunk'], d['config']['kary_mode'], d['clocks']['sm_mhz'], d['parity_sample_ok'])"
timeout 600 python bench.py --config config2 --no-e2e > gpurun_out/s3y_bench_config2.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s3y_bench_config2.json'));print('c2', round(d['value']/1e9,2), d['config']['leaf_chunk'], d['config']['kary_mode'], d['clocks']['sm_mhz'], d['parity_sample_ok'], d.get('speedup_vs_naive'))"
timeout 1500 python tools/size_sweep.py --kb 4 --lo 15 --hi 29 --step 2 > gpurun_out/s3y_size_u32.jsonl 2> gpurun_out/s3y_size.err; echo "u32 rc=$?"
timeout 1500 python tools/size_sweep.py --kb 8 --lo 16 --hi 30 --step 2 > gpurun_out/s3y_size_u64.jsonl 2>> gpurun_out/s3y_size.err; echo "u64 rc=$?"; tail -2 gpurun_out/s3y_size.err
