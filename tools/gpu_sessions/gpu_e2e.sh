#!/bin/bash
# e2e (bs_lookup_host) vs the PCIe floor: chunk size / stage count knobs.
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for cfgk in "22 4" "24 4" "20 4" "22 2" "22 8" "23 3"; do
  set -- $cfgk
  BS_HOST_CHUNK_LOG2=$1 BS_HOST_STAGES=$2 timeout 600 python bench.py --steps 5 --warmup 3 --no-naive > $O/e2e_c$1_s$2.json 2> $O/e2e_c$1_s$2.err
  python -c "import json;d=json.loads(open('$O/e2e_c$1_s$2.json').read().strip().splitlines()[-1]);e=d['e2e'];print('chunk 2^$1 stages $2 e2e G/s',round(e['value']/1e9,3),'ms',round(e['ms_per_step'],2),'pcie floor ms',round(e['pcie_floor_ms'],2),'frac',round(e['frac_of_pcie_floor'],3),'| dev G/s',round(d['value']/1e9,2))"
done
