#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/probe3.log
for cfg in 3 4 2; do timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep -E "config|rror" >> gpurun_out/probe3.log; done
cat gpurun_out/probe3.log
