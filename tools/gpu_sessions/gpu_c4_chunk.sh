#!/bin/bash
# Config 4 (two-level BUCKET): search item size vs time and DRAM traffic of the search.
# usage: gpu_c4_chunk.sh TAG
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for CH in 8192 16384 32768 65536; do
  BS_BUCKET_CHUNK=$CH timeout 600 python bench.py --config config4 --steps 3 --warmup 3 --no-e2e --no-naive > $O/bench_ch$CH.json 2> $O/bench_ch$CH.err
  python -c "import json;d=json.loads(open('$O/bench_ch$CH.json').read().strip().splitlines()[-1]);print('CH $CH G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),'parity',d.get('parity_sample_ok'))"
  BS_BUCKET_CHUNK=$CH timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_bk_search -c 1 --csv --log-file $O/ncu_ch$CH.csv python bench.py --config config4 --steps 1 --warmup 3 --no-e2e --no-naive > /dev/null 2>&1
  python tools/ncu_kernels.py $O/ncu_ch$CH.csv --per 1073741824
done
