#!/bin/bash
mkdir -p gpurun_out
for c in 1 2 3 4 5; do
  timeout 1200 python bench.py --config $c > gpurun_out/bench_full_cfg$c.log 2>&1; echo "cfg$c rc=$?" >> gpurun_out/bench_full_cfg$c.log
  tail -1 gpurun_out/bench_full_cfg$c.log
done
