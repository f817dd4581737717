#!/bin/bash
# factorization batch size sweep (SLIM_BATCH) over configurations
set -u
mkdir -p gpurun_out
for c in ${CONFIGS:-2}; do
  for D in ${DS:-8 12 16}; do
    log=gpurun_out/bsweep_${c}_${D}.log
    SLIM_BATCH=$D timeout 900 python bench.py --config $c --quick --steps ${STEPS:-48} > $log 2>&1
    grep '^{' $log | tail -1 | python -c "
import json,sys
s=sys.stdin.read().strip()
if not s: print('cfg $c D=$D FAILED'); sys.exit()
d=json.loads(s); print('cfg $c D=$D', round(d['value'],1), 'it/s', {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3))"
  done
done
