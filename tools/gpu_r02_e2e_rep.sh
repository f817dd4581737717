#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2 3 4; do
  SLIM_TRACE_RUN=1 timeout 600 python tools/e2e_trace.py 3 32 > gpurun_out/e2e_rep_$i.log 2>&1
  grep "^rep " gpurun_out/e2e_rep_$i.log
done
