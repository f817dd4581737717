#!/bin/bash
# round profiles: one steady-state k_chol_tiles capture per configuration
# (ncu --set full) and the launch list of the default bench command
set -u
mkdir -p gpurun_out
for spec in "2 32 2" "3 24 6" "5 32 2"; do
  set -- $spec
  CMD="python bench.py --config $1 --steps $2 --warmup 3 --quick"
  timeout 900 $CMD > gpurun_out/prof_plain_cfg$1.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_chol_tiles -s $3 -c 1 \
    -o gpurun_out/chol_full_cfg$1 $CMD > gpurun_out/prof_ncu_cfg$1.log 2>&1
  echo "cfg$1 capture rc=$?"
done
CMD="python bench.py --steps 16 --warmup 3 --quick"
timeout 600 $CMD > gpurun_out/list_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/list_ncu.log 2>&1
echo "list rc=$?"
