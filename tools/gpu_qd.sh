#!/bin/bash
# digit count A/B: QD=8 (default build) vs QD=7 (libslimb200_qd7.so): parity suite + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_qd8.log 2>&1; echo "qd8 rc=$?"; tail -2 gpurun_out/pytest_qd8.log
SLIM_LIB=$PWD/paper_1912_07962_b200/libslimb200_qd7.so timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_qd7.log 2>&1; echo "qd7 rc=$?"; tail -4 gpurun_out/pytest_qd7.log
for v in 8 7; do
  if [ $v = 7 ]; then export SLIM_LIB=$PWD/paper_1912_07962_b200/libslimb200_qd7.so; else unset SLIM_LIB; fi
  for c in 2 3 4; do
    timeout 600 python bench.py --bare --config $c > gpurun_out/qd${v}_$c.log 2>&1
    python -c "
import json
for ln in open('gpurun_out/qd${v}_$c.log'):
    if ln.startswith('{'):
        d=json.loads(ln); print('QD=$v cfg$c', round(d['value'],2), d['kernel_ms_per_step'], 'fp64eq', round(d['roofline']['fp64_equivalent_tflops'],1), 'err', d['final_rel_err_x_true'])
"
  done
done
