#!/bin/bash
# round-2 validation: the whole -m gpu suite, smoke, then both bench arms as the driver runs them
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -rA > gpurun_out/full_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/full_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref.out 2> gpurun_out/ref.err
echo "ref rc=$?" >> gpurun_out/ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.out 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/full_suite.log gpurun_out/smoke.log gpurun_out/ref.err gpurun_out/bench.err
