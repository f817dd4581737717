#!/bin/bash
# k_chol_i8 at 2 CTAs per SM (NST=2, 128 registers) vs the default build
mkdir -p gpurun_out
ALT=$PWD/paper_1912_07962_b200/libslimb200_occ2.so
SLIM_LIB=$ALT timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config or tomo or potrf" > gpurun_out/pytest_occ2.log 2>&1; echo "occ2 tests rc=$?"; tail -2 gpurun_out/pytest_occ2.log
for v in base occ2; do
  if [ $v = occ2 ]; then export SLIM_LIB=$ALT; else unset SLIM_LIB; fi
  for c in 2 3 5; do
    timeout 600 python bench.py --bare --config $c > gpurun_out/occ_${v}_$c.log 2>&1
    python -c "
import json
for ln in open('gpurun_out/occ_${v}_$c.log'):
    if ln.startswith('{'):
        d=json.loads(ln); print('$v cfg$c', round(d['value'],2), d['kernel_ms_per_step'])
" || tail -3 gpurun_out/occ_${v}_$c.log
  done
done
