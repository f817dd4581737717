#!/bin/bash
# GPU suite (incl. the digit-layout test) + accumulator back-off 250 ns
# (libslimb200_s250.so) and 12-system batches at configs[1]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu2.log
run() {  # tag config [env...]
  local tag=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --bare --config $c > gpurun_out/knob2_${tag}_$c.log 2>&1
  python -c "
import json
for ln in open('gpurun_out/knob2_${tag}_$c.log'):
    if ln.startswith('{'):
        d=json.loads(ln); print('$tag cfg$c', round(d['value'],2), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})
"
}
S250=SLIM_LIB=$PWD/paper_1912_07962_b200/libslimb200_s250.so
for rep in 1 2; do run base 2 A=1; run s250 2 $S250; run b12 2 SLIM_BATCH=12; done
run base 3 A=1; run s250 3 $S250
