#!/bin/bash
# A/B of an environment switch on one configuration: VAR=name VALS="a b" CFG=2 REPS=2
set -u
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do
  for v in ${VALS}; do
    env $VAR=$v timeout 600 python bench.py --config ${CFG:-2} --quick --steps ${STEPS:-48} 2>&1 | grep '^{' | tail -1 | python -c "
import json,sys
s=sys.stdin.read().strip()
if not s: print('$VAR=$v FAILED'); sys.exit()
d=json.loads(s); print('$VAR=$v', round(d['value'],1), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
  done
done
