#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/chol_order_sweep.py --config 3 --orders 1:32,2:16,2:32,3:32,4:32,4:64 --repeat 2 > gpurun_out/band64.log 2>&1
timeout 900 python tools/chol_order_sweep.py --config 2 --steps 176 --orders 1:32,2:16,4:32 --repeat 2 >> gpurun_out/band64.log 2>&1
timeout 900 python tools/chol_order_sweep.py --config 4 --steps 48 --orders 1:32,2:16,4:32 --repeat 1 >> gpurun_out/band64.log 2>&1
grep rep gpurun_out/band64.log
