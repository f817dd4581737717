#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "refinement or refined or fixed_point" > gpurun_out/new_tests.log 2>&1
echo "rc=$?" >> gpurun_out/new_tests.log
tail -n 12 gpurun_out/new_tests.log | cut -c1-200
