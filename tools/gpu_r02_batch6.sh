#!/bin/bash
# systems per factorization launch (SLIM_BATCH) with the six-digit, three-stage kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/batch6.log
for d in 2 3 4 5; do
  echo "== SLIM_BATCH=$d" >> gpurun_out/batch6.log
  SLIM_BATCH=$d timeout 600 python tools/chol_order_sweep.py --config 3 --steps 48 --orders 1:32 --repeat 1 2>&1 | grep -E "rep|rror" >> gpurun_out/batch6.log
  SLIM_BATCH=$d timeout 600 python tools/chol_order_sweep.py --config 4 --steps 48 --orders 1:32 --repeat 1 2>&1 | grep -E "rep|rror" >> gpurun_out/batch6.log
done
cat gpurun_out/batch6.log
