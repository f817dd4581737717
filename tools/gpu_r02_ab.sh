#!/bin/bash
# same-box A/B of library variants: VARIANTS="default head b3" (libslimb200_<tag>.so)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_1912_07962_b200
for rep in 1 2; do
for v in ${VARIANTS:-default head}; do
  if [ $v = default ]; then unset SLIM_LIB; else export SLIM_LIB=$L/libslimb200_$v.so; fi
  echo "== $v" >> gpurun_out/ab.log
  timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 1 2>&1 | grep rep >> gpurun_out/ab.log
  timeout 600 python tools/chol_order_sweep.py --config 2 --steps 176 --orders 1:32 --repeat 1 2>&1 | grep rep >> gpurun_out/ab.log
done
done
cat gpurun_out/ab.log
