#!/bin/bash
# factorization time vs operand bytes: the default kernel and one that loads
# every stage's B box twice (+1/3 of the operand bytes), configs[2] and [1]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_1912_07962_b200
for v in default extrab default extrab; do
  if [ $v = extrab ]; then export SLIM_LIB=$L/libslimb200_extrab.so; else unset SLIM_LIB; fi
  echo "== $v" >> gpurun_out/extrab.log
  timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 1 2>&1 | grep rep >> gpurun_out/extrab.log
  timeout 600 python tools/chol_order_sweep.py --config 2 --steps 96 --orders 1:32 --repeat 1 2>&1 | grep rep >> gpurun_out/extrab.log
done
cat gpurun_out/extrab.log
