#!/bin/bash
# device timeline of the bench's e2e run (public run() on a fresh host operator)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
SLIM_TRACE_RUN=1 timeout 600 python tools/e2e_trace.py ${CFG:-3} ${TOTAL:-32} > gpurun_out/e2e_trace_cfg${CFG:-3}.log 2>&1
tail -n 40 gpurun_out/e2e_trace_cfg${CFG:-3}.log
