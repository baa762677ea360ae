#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2aj}
mkdir -p $O
for T in 1 2; do
BS_BUCKET_T=$T timeout 600 python bench.py --config config4 --reorder 5 --steps 3 --no-e2e --no-naive > $O/bench_c4_T$T.json 2> $O/bench_c4_T$T.err
python -c "import json;d=json.loads(open('$O/bench_c4_T$T.json').read().strip().splitlines()[-1]);print('c4 T$T G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
BS_BUCKET_T=$T BS_BUCKET_COARSE=1 timeout 300 python bench.py --reorder 5 --no-e2e --no-naive > $O/bench_c3c_T$T.json 2> $O/bench_c3c_T$T.err
python -c "import json;d=json.loads(open('$O/bench_c3c_T$T.json').read().strip().splitlines()[-1]);print('c3 coarse T$T G/s',d['value']/1e9,'ms',d['ms_per_step'],d['parity_sample_ok'],d['invariant_all_ok'])"
done
