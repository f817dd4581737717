#!/bin/bash
# per-kernel launch list (ncu, isolated launches) of one bench configuration
set -u
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-2} --steps ${STEPS:-16} --warmup 3 --bare"
timeout 600 $CMD > gpurun_out/plain_cfg${CFG:-2}.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/plain_cfg${CFG:-2}.log | cut -c1-300
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-2000} --csv \
  --log-file gpurun_out/launches_cfg${CFG:-2}.csv $CMD > gpurun_out/ncu_list_cfg${CFG:-2}.log 2>&1
echo "list rc=$?"
