#!/bin/bash
# split operand rings: A 3 deep + B 2 deep (default) vs 2 + 2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_1912_07962_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_runs.py -m gpu -q -s -x \
  -k "potrf or dense_runs or digit_layout or config1_one_epoch or large_tomography or tomo_runs or sharded" \
  > gpurun_out/rings_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rings_tests.log
for v in a3b2 a2b2 a3b2 a2b2; do
  if [ $v = a2b2 ]; then export SLIM_LIB=$L/libslimb200_b3.so; else unset SLIM_LIB; fi
  echo "== $v" >> gpurun_out/rings_speed.log
  timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 1 2>&1 | grep rep >> gpurun_out/rings_speed.log
  timeout 600 python tools/chol_order_sweep.py --config 2 --steps 176 --orders 1:32 --repeat 1 2>&1 | grep rep >> gpurun_out/rings_speed.log
done
grep -E "relative|passed|failed|rc=" gpurun_out/rings_tests.log; cat gpurun_out/rings_speed.log
