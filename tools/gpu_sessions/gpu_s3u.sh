#!/bin/bash
# kary_mode 6 vs 7: sustained bench lines on configs 3 and 2, alternating
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for md in 6 7; do
  timeout 600 python bench.py --no-e2e --no-naive --kary-mode $md --steps 100 > gpurun_out/s3u_c3_m${md}_r$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/s3u_c3_m${md}_r$rep.json'));print('config3 mode $md rep $rep', round(d['value']/1e9,2), d['clocks']['sm_mhz'], d['parity_sample_ok'])"
done
done
for md in 6 7; do
  timeout 600 python bench.py --config config2 --no-e2e --no-naive --kary-mode $md --steps 100 > gpurun_out/s3u_c2_m${md}.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/s3u_c2_m${md}.json'));print('config2 mode $md', round(d['value']/1e9,2), d['clocks']['sm_mhz'], d['parity_sample_ok'])"
done
