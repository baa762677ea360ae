#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2bs}
mkdir -p $O
run() { local name=$1; shift; env "$@" timeout 600 python bench.py --steps 5 --no-e2e --no-naive $BA > $O/$name.json 2>/dev/null; python -c "import json;d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]);print('$name G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),d['parity_sample_ok'],d['invariant_all_ok'])"; }
BA="" run c3_two BS_BUCKET_TWO=1
BA="--config config4" run c4_ch16k BS_BUCKET_CHUNK=16384
BA="--config config4" run c4_ch32k BS_BUCKET_CHUNK=32768
BA="--config config4" run c4_default X=1
BA="--config config4 --reorder 5" run c4_g8 BS_BUCKET_G8=1
