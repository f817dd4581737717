#!/bin/bash
# round-2 session-4 baseline: -m gpu suite, smoke, default bench, e2e phase split at configs[2] and configs[1]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/s4_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s4_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4_bench.out 2> gpurun_out/s4_bench.err
echo "bench rc=$?" >> gpurun_out/s4_bench.err
timeout 600 python tools/e2e_phases.py 3 > gpurun_out/s4_e2e_cfg3.log 2>&1
timeout 600 python tools/e2e_phases.py 2 > gpurun_out/s4_e2e_cfg2.log 2>&1
tail -3 gpurun_out/s4_suite.log gpurun_out/s4_smoke.log gpurun_out/s4_bench.err gpurun_out/s4_e2e_cfg3.log
