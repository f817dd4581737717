#!/bin/bash
# after ordering the task-map upload on the factorization stream: shard stress, sharded tests, default bench, e2e trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/close_shards.log
for P in 3 4 3 4; do timeout 200 python tools/shard_stress.py 400 $P 2>&1 | grep -v "^  " | tail -n 1 >> gpurun_out/close_shards.log; done
for i in 1 2 3; do timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sharded" 2>&1 | tail -n 1 >> gpurun_out/close_shards.log; done
cat gpurun_out/close_shards.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/close_bench.out 2> gpurun_out/close_bench.err
echo "bench rc=$?" >> gpurun_out/close_bench.err
tail -n 2 gpurun_out/close_bench.err
SLIM_TRACE_RUN=1 timeout 600 python tools/e2e_trace.py 3 32 2>&1 | grep "^rep "
