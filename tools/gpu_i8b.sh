# int8 factorization: accuracy, GPU parity suite, bench A/B vs DMMA
mkdir -p gpurun_out
SLIM_CHOL=i8 timeout 300 python tools/chol_check.py 600 3982 8000 13032 > gpurun_out/i8.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 2 3 4 5 1; do VAR=SLIM_CHOL VALS="dmma i8" CFG=$c REPS=1 STEPS=${STEPS:-48} bash tools/gpu_ab.sh >> gpurun_out/i8.log 2>&1; done
cat gpurun_out/i8.log; tail -15 gpurun_out/pytest_gpu.log
