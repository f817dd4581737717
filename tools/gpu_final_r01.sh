#!/bin/bash
# end-of-round evidence: GPU suite, smoke, full bench lines for every config,
# the reference arm, the bare launch list of the headline config
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 1 3 4 5; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_full_cfg$c.log 2>&1; echo "cfg$c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CFG=2 bash tools/gpu_launches.sh
