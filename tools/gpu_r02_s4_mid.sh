#!/bin/bash
# validation after the upload-path fix: -m gpu suite, default bench, configs[1] bench, e2e trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/s4_suite.log
tail -n 3 gpurun_out/s4_suite.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4_bench.out 2> gpurun_out/s4_bench.err
echo "bench rc=$?" >> gpurun_out/s4_bench.err
tail -n 2 gpurun_out/s4_bench.err
timeout 900 python bench.py --config 2 --gpus 1 --steps 176 --warmup 5 > gpurun_out/s4_bench_cfg2.out 2> gpurun_out/s4_bench_cfg2.err
echo "bench rc=$?" >> gpurun_out/s4_bench_cfg2.err
tail -n 2 gpurun_out/s4_bench_cfg2.err
SLIM_TRACE_RUN=1 timeout 600 python tools/e2e_trace.py 2 192 > gpurun_out/e2e_trace_cfg2.log 2>&1
grep "rep " gpurun_out/e2e_trace_cfg2.log
