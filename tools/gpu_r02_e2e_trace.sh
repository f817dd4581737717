#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
SLIM_TRACE_RUN=1 timeout 600 python tools/e2e_trace.py 3 32 > gpurun_out/e2e_trace_cfg3.log 2>&1
tail -n 40 gpurun_out/e2e_trace_cfg3.log
