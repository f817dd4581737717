#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for q in 0 1 2 3 4 5; do
  SLIM_MTW_QUAD=$q timeout 300 python tools/stream_probe.py --config 3 2>&1 | grep config >> gpurun_out/mtw_probe.log
done
for q in 0 2 3; do
  SLIM_MTW_QUAD=$q timeout 300 python tools/stream_probe.py --config 2 2>&1 | grep config >> gpurun_out/mtw_probe.log
  SLIM_MTW_QUAD=$q timeout 300 python tools/stream_probe.py --config 4 2>&1 | grep config >> gpurun_out/mtw_probe.log
done
cat gpurun_out/mtw_probe.log
