#!/bin/bash
# run-to-run spread of the headline (fresh process each time, the driver's invocation without the side legs)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/variance.log
for i in 1 2 3 4 5 6 7 8; do
  timeout 300 python bench.py --steps 20 --warmup 5 --bare 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],2), round(d['ms_per_step'],3), d['kernel_ms_per_step'], d['clocks'])" >> gpurun_out/variance.log
done
cat gpurun_out/variance.log
