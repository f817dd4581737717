#!/bin/bash
# round profile set: GPU tests, smoke, default bench line (configs[1]), the other
# configs, the reference arm, launch list, steady-state ncu of the factorization
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"
for c in 1 3 4 5; do timeout 900 python bench.py --config $c > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"; done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CFG=2 STEPS=16 bash tools/gpu_launches.sh
CS="2:3 3:5" bash tools/gpu_ncu_steady.sh
