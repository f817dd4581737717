# quick iteration: potrf accuracy, GPU parity, bench A/B, trace
mkdir -p gpurun_out
timeout 300 python tools/chol_check.py 600 3982 13032 > gpurun_out/it.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/it.log
for c in ${CFGS:-2 3}; do VAR=${VAR:-SLIM_BATCH} VALS="${VALS:-16}" CFG=$c REPS=1 STEPS=${STEPS:-48} bash tools/gpu_ab.sh >> gpurun_out/it.log 2>&1; done
CFG=2 bash tools/gpu_trace_i8.sh >> gpurun_out/it.log 2>&1
cat gpurun_out/it.log
