#!/bin/bash
# speed of the factorization with fewer digits (upper bound on what refinement could buy)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_1912_07962_b200
: > gpurun_out/digits6_speed.log
for v in default qd6x1 qd6x0 qd5x1; do
  if [ $v = default ]; then unset SLIM_LIB; else export SLIM_LIB=$L/libslimb200_$v.so; fi
  echo "== $v" >> gpurun_out/digits6_speed.log
  timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 2 2>&1 | grep -E "rep|rror" >> gpurun_out/digits6_speed.log
  timeout 600 python tools/chol_order_sweep.py --config 2 --steps 176 --orders 1:32 --repeat 1 2>&1 | grep -E "rep|rror" >> gpurun_out/digits6_speed.log
done
cat gpurun_out/digits6_speed.log
