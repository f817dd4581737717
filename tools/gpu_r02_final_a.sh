#!/bin/bash
# round-2 final validation, part A: the whole -m gpu suite and smoke
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -rA > gpurun_out/final_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/final_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
tail -n 3 gpurun_out/final_suite.log | cut -c1-200; tail -n 2 gpurun_out/final_smoke.log
