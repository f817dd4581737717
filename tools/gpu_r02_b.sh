#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_full_runs.py tests/test_gpu_stream_file.py tests/test_gpu_contract.py -m gpu -q -s \
  -k "config1_one_epoch or stream" > gpurun_out/b_tests.log 2>&1
echo "rc=$?" >> gpurun_out/b_tests.log
timeout 1500 python tools/chol_order_sweep.py --config 3 --orders 1:32,2:16,2:32,3:32,4:32,4:64 > gpurun_out/order3.log 2>&1
timeout 900 python tools/chol_order_sweep.py --config 2 --steps 96 --orders 1:32,2:16,2:32,3:32,4:32 > gpurun_out/order2.log 2>&1
tail -3 gpurun_out/b_tests.log; cat gpurun_out/order3.log gpurun_out/order2.log | grep rep
