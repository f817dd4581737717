#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 ./tools/microbench/tma_rows > gpurun_out/tma_rows.log 2>&1
timeout 900 python tools/race_stress.py --config 2 --steps 64 --reps 12 --oracle > gpurun_out/stress.log 2>&1
timeout 900 python tools/race_stress.py --config 1 --steps 200 --reps 12 >> gpurun_out/stress.log 2>&1
timeout 900 python tools/race_stress.py --config 3 --steps 20 --reps 4 >> gpurun_out/stress.log 2>&1
cat gpurun_out/tma_rows.log; grep -E "differing|oracle" gpurun_out/stress.log
