#!/bin/bash
# round-2 closing check on the final tree: -m gpu suite, smoke, both bench arms as the driver runs them,
# the sharded selection repeated, a last shard stress
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -rA > gpurun_out/final_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/final_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/close_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/close_smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/close_ref.out 2> gpurun_out/close_ref.err
echo "ref rc=$?" >> gpurun_out/close_ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/close_bench.out 2> gpurun_out/close_bench.err
echo "bench rc=$?" >> gpurun_out/close_bench.err
timeout 900 python bench.py --config 2 --gpus 1 --steps 176 --warmup 5 > gpurun_out/close_bench_cfg2.out 2> gpurun_out/close_bench_cfg2.err
echo "bench cfg2 rc=$?" >> gpurun_out/close_bench_cfg2.err
: > gpurun_out/close_shards.log
for i in 1 2 3 4 5 6; do timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sharded" 2>&1 | tail -n 1 >> gpurun_out/close_shards.log; done
for P in 3 4; do timeout 200 python tools/shard_stress.py 400 $P 2>&1 | grep -v "^  " | tail -n 1 >> gpurun_out/close_shards.log; done
tail -n 3 gpurun_out/final_suite.log | cut -c1-150; tail -n 2 gpurun_out/close_smoke.log; tail -n 1 gpurun_out/close_ref.err gpurun_out/close_bench.err gpurun_out/close_bench_cfg2.err; cat gpurun_out/close_shards.log
