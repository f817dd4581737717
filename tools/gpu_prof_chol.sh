#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps ${STEPS:-32} --warmup 3 --quick --config ${CFG:-2}"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_chol_i8} -s ${SKIP:-2} -c 1 -o gpurun_out/chol_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
