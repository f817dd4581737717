#!/bin/bash
# six-digit factorization with a three-stage operand ring (3 x 72 KB = 217 KB) vs two stages
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_1912_07962_b200
: > gpurun_out/nst3.log
for v in default q6nst3; do
  if [ $v = default ]; then unset SLIM_LIB; else export SLIM_LIB=$L/libslimb200_$v.so; fi
  echo "== $v" >> gpurun_out/nst3.log
  timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 2 2>&1 | grep -E "rep|rror" >> gpurun_out/nst3.log
  timeout 600 python tools/chol_order_sweep.py --config 4 --orders 1:32 --repeat 1 2>&1 | grep -E "rep|rror" >> gpurun_out/nst3.log
done
cat gpurun_out/nst3.log
