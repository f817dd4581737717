#!/bin/bash
# ticket order A/B with the six-digit factorization (more DRAM-bound than seven digits)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/chol_order_sweep.py --config 3 --orders 1:32,2:16,2:32,3:32,4:32 --repeat 2 2>&1 | grep -E "rep|rror" > gpurun_out/order6_cfg3.log
timeout 900 python tools/chol_order_sweep.py --config 4 --orders 1:32,2:16,2:32,3:32 --repeat 1 2>&1 | grep -E "rep|rror" > gpurun_out/order6_cfg4.log
cat gpurun_out/order6_cfg3.log gpurun_out/order6_cfg4.log
