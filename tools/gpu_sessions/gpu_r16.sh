#!/bin/bash
# Two-level search: lookups in flight per thread (BS_BUCKET_R16 = 0 (2 @ 768 thr), 3 @ 640, 4 @ 512), config 4 and 5.
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for rep in 1 2; do
for R in 0 3 4; do
  BS_BUCKET_R16=$R timeout 600 python bench.py --config config4 --steps 5 --warmup 3 --no-e2e --no-naive > $O/c4_R${R}_$rep.json 2> $O/c4_R${R}_$rep.err
  python -c "import json;d=json.loads(open('$O/c4_R${R}_$rep.json').read().strip().splitlines()[-1]);print('c4 R16=$R rep $rep G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),'parity',d.get('parity_sample_ok'))"
done; done
for R in 0 3 4; do
  BS_BUCKET_R16=$R timeout 600 python bench.py --config config5 --steps 5 --warmup 3 --no-e2e --no-naive --no-dist > $O/c5_R${R}.json 2> $O/c5_R${R}.err
  python -c "import json;d=json.loads(open('$O/c5_R${R}.json').read().strip().splitlines()[-1]);print('c5 R16=$R G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),'parity',d.get('parity_sample_ok'))"
done
