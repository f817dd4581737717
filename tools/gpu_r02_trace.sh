#!/bin/bash
# per-task phase timeline of one steady factorization launch (globaltimer stamps)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for cfg in 3 2; do
  TL=$([ $cfg = 3 ] && echo 9 || echo 4)
  SLIM_CHOL_TRACE=gpurun_out/trace_cfg$cfg.csv SLIM_CHOL_TRACE_LAUNCH=$TL timeout 600 \
    python bench.py --config $cfg --steps 32 --warmup 3 --bare > gpurun_out/trace_bench$cfg.log 2>&1
  echo "== config $cfg launch $TL" >> gpurun_out/trace_phases.log
  python tools/trace_phases.py gpurun_out/trace_cfg$cfg.csv >> gpurun_out/trace_phases.log 2>&1
done
cat gpurun_out/trace_phases.log
