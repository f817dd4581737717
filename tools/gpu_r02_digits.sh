#!/bin/bash
# parity margin and speed of the factorization's digit layouts (round 2)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_1912_07962_b200
for v in default qx1 qd8 dmma; do
  case $v in
    default) envs="";;
    dmma) envs="SLIM_CHOL=dmma";;
    *) envs="SLIM_LIB=$PWD/$L/libslimb200_$v.so";;
  esac
  echo "== $v" >> gpurun_out/digits.log
  env $envs timeout 900 python -m pytest tests/test_gpu_full_runs.py -m gpu -q -s \
    -k "config1_one_epoch or large_tomography" 2>&1 | grep -E "relative|passed|failed" >> gpurun_out/digits.log
done
for v in default qx1 qd8 dmma; do
  case $v in
    default) envs="";;
    dmma) envs="SLIM_CHOL=dmma";;
    *) envs="SLIM_LIB=$PWD/$L/libslimb200_$v.so";;
  esac
  echo "== $v" >> gpurun_out/digits_speed.log
  env $envs timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 2 2>&1 | grep rep >> gpurun_out/digits_speed.log
  env $envs timeout 600 python tools/chol_order_sweep.py --config 2 --steps 176 --orders 1:32 --repeat 2 2>&1 | grep rep >> gpurun_out/digits_speed.log
done
cat gpurun_out/digits.log gpurun_out/digits_speed.log
