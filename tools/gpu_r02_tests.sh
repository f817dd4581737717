#!/bin/bash
# round-2 GPU check: new contract / full-run tests, then the whole -m gpu suite
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_contract.py tests/test_gpu_full_runs.py -m gpu -q -s \
  -k "${SEL:-contract or config0 or config4}" > gpurun_out/new_tests.log 2>&1
echo "new_tests rc=$?" >> gpurun_out/new_tests.log
timeout 1500 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_full_runs.py \
  --ignore=tests/test_gpu_contract.py > gpurun_out/suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/suite.log
tail -3 gpurun_out/new_tests.log gpurun_out/suite.log
