#!/bin/bash
# knob A/B with the 7-digit (8-bit trailing) factorization: TMA ring depth 4
# (libslimb200_nst4.so) and batch size for the N > 6144 configurations
mkdir -p gpurun_out
timeout 600 python tools/parity_margins.py > gpurun_out/margins_d8.log 2>&1; cat gpurun_out/margins_d8.log
SLIM_LIB=$PWD/paper_1912_07962_b200/libslimb200_d7.so timeout 600 python tools/parity_margins.py > gpurun_out/margins_d7.log 2>&1; cat gpurun_out/margins_d7.log
run() {  # tag config [env...]
  local tag=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --bare --config $c > gpurun_out/knob_${tag}_$c.log 2>&1
  python -c "
import json
for ln in open('gpurun_out/knob_${tag}_$c.log'):
    if ln.startswith('{'):
        d=json.loads(ln); print('$tag cfg$c', round(d['value'],2), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})
"
}
NST4=SLIM_LIB=$PWD/paper_1912_07962_b200/libslimb200_nst4.so
run base 2 A=1; run nst4 2 $NST4; run base 2 A=1; run nst4 2 $NST4
run base 3 A=1; run nst4 3 $NST4; run b6 3 SLIM_BATCH=6; run b8 3 SLIM_BATCH=8
run base 4 A=1; run b6 4 SLIM_BATCH=6; run b8 4 SLIM_BATCH=8
