#!/bin/bash
# A/B timing of two library builds (lib/libbs_A.so, lib/libbs_B.so), interleaved.  usage: gpu_ab.sh TAG [bench args]
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for rep in 1 2 3; do
for v in A B; do
BS_LIB_PATH=$PWD/paper_2506_01576_b200/lib/libbs_$v.so timeout 300 python bench.py --steps 20 --no-e2e --no-naive "$@" > $O/b_${v}_$rep.json 2>/dev/null
python -c "import json;d=json.loads(open('$O/b_${v}_$rep.json').read().strip().splitlines()[-1]);print('$v rep $rep G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],4),d['parity_sample_ok'],d['invariant_all_ok'])"
done
done
