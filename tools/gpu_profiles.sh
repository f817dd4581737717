#!/bin/bash
# round profile set: default bench line (configs[1]), other configs, launch list,
# ncu --set full of the factorization at configs[1] and configs[2]
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"
for c in 1 3 4 5; do timeout 900 python bench.py --config $c > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"; done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CFG=2 STEPS=16 bash tools/gpu_launches.sh
for c in 2 3; do
  CMD="python bench.py --steps 32 --warmup 3 --quick --config $c"
  timeout 600 $CMD > gpurun_out/plain_p$c.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_chol_i8 -s 2 -c 1 -o gpurun_out/chol_full_cfg$c $CMD > gpurun_out/ncu_full_cfg$c.log 2>&1
  echo "ncu cfg$c rc=$?"
done
