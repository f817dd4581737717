#!/bin/bash
# ncu --set full of one steady-state k_chol_i8 launch at configs[2] (4 systems
# of N = 13,032): launches 1-3 are the bench's warm-up run (k = 1..10), 4-6 the
# timed run's warm-up batches; launch 9 (k = 21..24) has a full window and
# tile reuse like every timed launch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --config 3 --steps 16 --warmup 3 --bare"
$CMD > gpurun_out/ncu_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_chol_i8 -s 8 -c 1 \
    -o gpurun_out/chol_cfg3_r02 $CMD > gpurun_out/ncu_chol.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_chol.log
tail -5 gpurun_out/ncu_chol.log
