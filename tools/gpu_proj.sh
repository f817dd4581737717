#!/bin/bash
# device projector tests, streaming probe A/B of the M^T w window grouping, full GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_projector.py -m gpu -x -q > gpurun_out/pytest_proj.log 2>&1; echo "proj rc=$?" >> gpurun_out/pytest_proj.log
tail -15 gpurun_out/pytest_proj.log
for g in 1 3 6; do
  SLIM_MTW_GROUP=$g CONFIGS="3 4 2" bash tools/gpu_stream.sh 2>&1 | sed "s/^/g$g /"
done
CONFIGS="1 5" bash tools/gpu_stream.sh
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
