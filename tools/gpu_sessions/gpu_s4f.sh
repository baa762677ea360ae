#!/bin/bash
# A/B: g1 FLAT T=1 instance with the output width as a compile-time constant vs the runtime-width instance
set -u
mkdir -p gpurun_out
T=${TAG:-r1s4f}
timeout 1200 python -m pytest tests -m gpu -q -rf -x --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
for r in 1 2 3; do
  for ab in runtime const; do
    if [ $ab = runtime ]; then export BS_G1_RUNTIME_OB=1; else unset BS_G1_RUNTIME_OB; fi
    timeout 300 python tools/mode_sweep.py --kb 8 --lo 26 --hi 26 --modes 7 2>/dev/null | sed "s/^{/{\"ab\": \"$ab\", \"rep\": $r, /" >> gpurun_out/${T}_ab.jsonl
    timeout 300 python tools/mode_sweep.py --kb 4 --lo 20 --hi 20 --modes 7 2>/dev/null | sed "s/^{/{\"ab\": \"$ab\", \"rep\": $r, /" >> gpurun_out/${T}_ab.jsonl
  done
done
unset BS_G1_RUNTIME_OB
cat gpurun_out/${T}_ab.jsonl
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cat gpurun_out/${T}_bench.json
