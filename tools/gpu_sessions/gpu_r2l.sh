#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_seg.py -x -q -k global > $O/pytest_seg.log 2>&1; echo "seg rc=$?"
timeout 600 python bench.py --config config3 --reorder 4 --steps 20 --no-e2e --no-naive > $O/bench_config3_global.json 2> $O/bench_config3_global.err; echo "c3g rc=$?"
for f in 0.5 0.75 0.9; do
  BS_SEP_L2_FRAC=$f timeout 600 python bench.py --config config4 --steps 5 --no-e2e --no-naive > $O/bench_config4_frac$f.json 2> $O/bench_config4_frac$f.err; echo "c4 $f rc=$?"
done
python - > $O/gen28.log 2>&1 <<'PY'
import torch, sys
sys.path.insert(0, ".")
from workload import device as wd
for lg in (27, 28, 29):
    k = wd.gen_keys(1 << lg, 8, device="cuda")
    f = wd._flip(k)
    print(lg, k.numel(), "sorted", bool((f[1:] > f[:-1]).all().item()), flush=True)
PY
echo "gen rc=$?"
CMD="python bench.py --config config3 --reorder 4 --steps 1 --warmup 3 --no-e2e --no-naive"
$CMD > $O/plain_full.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_part$|^k_unpart$" -s 2 -c 2 -o $O/kpart $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
