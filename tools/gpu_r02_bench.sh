#!/bin/bash
# round-2: selected GPU tests, then the default bench (both arms) as the driver runs it
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
if [ -n "$SEL" ]; then
  timeout 1800 python -m pytest tests/test_gpu_contract.py tests/test_gpu_full_runs.py -m gpu -q -s \
    -k "$SEL" > gpurun_out/sel_tests.log 2>&1
  echo "sel rc=$?" >> gpurun_out/sel_tests.log
fi
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref.out 2> gpurun_out/ref.err
echo "ref rc=$?" >> gpurun_out/ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.out 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
tail -2 gpurun_out/sel_tests.log gpurun_out/ref.err gpurun_out/bench.err
