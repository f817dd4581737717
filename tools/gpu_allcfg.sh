#!/bin/bash
# full bench line (cpu_baseline, e2e) for every configuration + the reference arm
mkdir -p gpurun_out
for c in ${CONFIGS:-1 2 3 4 5}; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_full_cfg$c.log 2>&1; echo "cfg$c rc=$?" >> gpurun_out/bench_full_cfg$c.log
  tail -2 gpurun_out/bench_full_cfg$c.log | cut -c1-160
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-200
