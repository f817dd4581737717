#!/bin/bash
# ncu launch list (device time of every kernel launch) of the bench's timed workload
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --config 3 --steps 16 --warmup 3 --bare"
$CMD > gpurun_out/launch_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_cfg3_r02.csv $CMD > gpurun_out/launch_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/launch_ncu.log
tail -3 gpurun_out/launch_ncu.log; wc -l gpurun_out/launches_cfg3_r02.csv
