#!/bin/bash
# quick iteration: chol trace, GPU tests, quick bench
mkdir -p gpurun_out
timeout 300 python tools/chol_trace.py 3982 > gpurun_out/trace.log 2>&1; echo "trace rc=$?" >> gpurun_out/trace.log
timeout 300 python tools/chol_trace.py 600 >> gpurun_out/trace.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --quick ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
cat gpurun_out/trace.log; tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-1500
