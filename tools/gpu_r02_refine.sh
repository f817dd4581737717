#!/bin/bash
# six-digit factorization + one refinement step of w (default for N > 6144) vs seven digits:
# parity of the full-size runs, then speed
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/refine.log
: > $out
for v in 1 0; do
  echo "== SLIM_REFINE=$v" >> $out
  SLIM_REFINE=$v timeout 900 python -m pytest tests/test_gpu_full_runs.py -m gpu -q -s 2>&1 | grep -E "relative|passed|failed|rror" >> $out
done
for v in 1 0; do
  echo "== SLIM_REFINE=$v speed" >> $out
  SLIM_REFINE=$v timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 2 2>&1 | grep -E "rep|rror" >> $out
  SLIM_REFINE=$v timeout 600 python tools/chol_order_sweep.py --config 4 --orders 1:32 --repeat 1 2>&1 | grep -E "rep|rror" >> $out
done
cat $out
