#!/bin/bash
# round-2 closing check on the final tree: -m gpu suite, smoke, both bench arms as the driver runs them, e2e timeline
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/close_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/close_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/close_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/close_smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/close_ref.out 2> gpurun_out/close_ref.err
echo "ref rc=$?" >> gpurun_out/close_ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/close_bench.out 2> gpurun_out/close_bench.err
echo "bench rc=$?" >> gpurun_out/close_bench.err
SLIM_TRACE_RUN=1 timeout 600 python tools/e2e_trace.py 3 32 > gpurun_out/e2e_trace_cfg3.log 2>&1
tail -n 3 gpurun_out/close_suite.log; tail -n 2 gpurun_out/close_smoke.log; tail -n 1 gpurun_out/close_ref.err gpurun_out/close_bench.err
