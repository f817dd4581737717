#!/bin/bash
# validation: ticket order A/B with the 3-stage six-digit kernel, -m gpu suite, default bench, configs[3] bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/chol_order_sweep.py --config 3 --orders 1:32,2:16,2:32 --repeat 2 2>&1 | grep -E "rep|rror" > gpurun_out/order6_nst3_cfg3.log
cat gpurun_out/order6_nst3_cfg3.log
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/s4_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/s4_suite.log
tail -n 3 gpurun_out/s4_suite.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4_bench.out 2> gpurun_out/s4_bench.err
echo "bench rc=$?" >> gpurun_out/s4_bench.err
tail -n 2 gpurun_out/s4_bench.err
timeout 900 python bench.py --config 4 --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4_bench_cfg4.out 2> gpurun_out/s4_bench_cfg4.err
echo "bench rc=$?" >> gpurun_out/s4_bench_cfg4.err
tail -n 2 gpurun_out/s4_bench_cfg4.err
