#!/bin/bash
# sorted-batch kernel with next-segment prefetch + 4 lookups per thread
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r2bb}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_seg.py -x -q > $O/pytest_seg.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_seg.log
for c in config3 config2; do
timeout 300 python bench.py --config $c --order sorted --no-e2e --no-naive > $O/b_$c.json 2>/dev/null
python -c "import json;d=json.loads(open('$O/b_$c.json').read().strip().splitlines()[-1]);print('$c sorted G/s',round(d['value']/1e9,2),'ms',round(d['ms_per_step'],3),d['parity_sample_ok'],d['invariant_all_ok'])"
done
