#!/bin/bash
# triangular-solve ring depth (32 KB slots of L tiles in flight per CTA): 3 (default) vs 4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/trsv_ring.log
for rs in 3 4; do
  echo "== SLIM_TRSV_RING=$rs" >> gpurun_out/trsv_ring.log
  SLIM_TRSV_RING=$rs timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 2 2>&1 | grep -E "rep|rror" >> gpurun_out/trsv_ring.log
  SLIM_TRSV_RING=$rs timeout 600 python tools/chol_order_sweep.py --config 4 --orders 1:32 --repeat 1 2>&1 | grep -E "rep|rror" >> gpurun_out/trsv_ring.log
  SLIM_TRSV_RING=$rs timeout 600 python tools/chol_order_sweep.py --config 2 --steps 176 --orders 1:32 --repeat 1 2>&1 | grep -E "rep|rror" >> gpurun_out/trsv_ring.log
done
cat gpurun_out/trsv_ring.log
