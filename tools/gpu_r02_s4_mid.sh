#!/bin/bash
# new streaming-kernel defaults: probe at configs[1..3], the whole -m gpu suite, default bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/stream_new_defaults.log
: > $out
for cfg in 3 2 4; do
  timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep -E "config|rror" >> $out
done
cat $out
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/s4_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/s4_suite.log
tail -n 3 gpurun_out/s4_suite.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4_bench.out 2> gpurun_out/s4_bench.err
echo "bench rc=$?" >> gpurun_out/s4_bench.err
tail -n 2 gpurun_out/s4_bench.err
