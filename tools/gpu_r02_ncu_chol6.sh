#!/bin/bash
# ncu --set full of one steady-state launch of the six-digit k_chol_i8 (slim::q6) at configs[2],
# plus the launch list of the same command
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --config 3 --steps 16 --warmup 3 --bare"
$CMD > gpurun_out/ncu_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_chol_i8 -s 8 -c 1 \
    -o gpurun_out/chol6_cfg3_r02 -f $CMD > gpurun_out/ncu_chol6.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_chol6.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg3_r02b.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
tail -n 3 gpurun_out/ncu_plain.log gpurun_out/ncu_chol6.log | cut -c1-300
