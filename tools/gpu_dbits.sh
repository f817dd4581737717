#!/bin/bash
# digit width A/B: default build (8 digits of 7 bits) vs libslimb200_d8.so
# (SLIM_QD=7 SLIM_DBITS=8: a 7-bit leading digit and six 8-bit digits, 55
# bits below the row scale, 28 digit pairs): parity suite + bench
mkdir -p gpurun_out
D8=$PWD/paper_1912_07962_b200/libslimb200_d8.so
SLIM_LIB=$D8 timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_d8.log 2>&1; echo "d8 rc=$?"; tail -4 gpurun_out/pytest_d8.log
for v in d8 d7; do
  if [ $v = d8 ]; then export SLIM_LIB=$D8; else unset SLIM_LIB; fi
  for c in ${CONFIGS:-2 3 4 5}; do
    timeout 600 python bench.py --bare --config $c > gpurun_out/${v}_$c.log 2>&1
    python -c "
import json
for ln in open('gpurun_out/${v}_$c.log'):
    if ln.startswith('{'):
        d=json.loads(ln); print('$v cfg$c', round(d['value'],2), d['kernel_ms_per_step'], 'fp64eq', round(d['roofline']['fp64_equivalent_tflops'],1), 'err', d['final_rel_err_x_true'])
"
  done
done
