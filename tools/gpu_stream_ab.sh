#!/bin/bash
# streaming kernels: M^T w staged (0) vs register-grouped (3); rowdot chunk counts
mkdir -p gpurun_out
for g in 0 3; do
  SLIM_MTW_GROUP=$g CONFIGS="3 2 4" bash tools/gpu_stream.sh 2>&1 | sed "s/^/mtw$g /"
done
for nch in; do
  SLIM_RD_NCH=$nch CONFIGS="5" bash tools/gpu_stream.sh 2>&1 | sed "s/^/nch$nch /"
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
