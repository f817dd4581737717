#!/bin/bash
# ncu --set full of one steady-state factorization launch per config
# (warm-up run + the timed run's first, from-scratch batch skipped)
mkdir -p gpurun_out
for cs in ${CS:-"2:3" "3:5"}; do
  c=${cs%%:*}; s=${cs##*:}
  CMD="python bench.py --steps 32 --warmup 3 --bare --config $c"
  timeout 600 $CMD > gpurun_out/plain_p$c.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_chol_i8 -s $s -c 1 -o gpurun_out/chol_full_cfg$c $CMD > gpurun_out/ncu_full_cfg$c.log 2>&1
  echo "ncu cfg$c rc=$?"
done
