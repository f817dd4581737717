#!/bin/bash
# launch list (isolated kernel times) + one full capture of the tile Cholesky
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 4 --warmup 3 --quick"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_chol_tiles -s 4 -c 1 -o gpurun_out/chol_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
