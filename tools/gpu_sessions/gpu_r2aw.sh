#!/bin/bash
# BUCKET knob sweep on config 3: search item size, table depth
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2aw}
mkdir -p $O
for CH in 8192 16384 32768 65536; do
BS_BUCKET_CHUNK=$CH timeout 300 python bench.py --steps 10 --no-e2e --no-naive > $O/b_ch$CH.json 2>/dev/null
python -c "import json;d=json.loads(open('$O/b_ch$CH.json').read().strip().splitlines()[-1]);print('CH $CH G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),d['parity_sample_ok'],d['invariant_all_ok'])"
done
BS_BUCKET_D=14 timeout 300 python bench.py --steps 10 --no-e2e --no-naive > $O/b_d14.json 2>/dev/null
python -c "import json;d=json.loads(open('$O/b_d14.json').read().strip().splitlines()[-1]);print('D14 G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),d['parity_sample_ok'],d['invariant_all_ok'])"
for CH in 16384 65536; do
BS_BUCKET_CHUNK=$CH timeout 600 python bench.py --config config4 --steps 3 --no-e2e --no-naive > $O/b4_ch$CH.json 2>/dev/null
python -c "import json;d=json.loads(open('$O/b4_ch$CH.json').read().strip().splitlines()[-1]);print('c4 CH $CH G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),d['parity_sample_ok'],d['invariant_all_ok'])"
done
