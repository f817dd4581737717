set -u
mkdir -p gpurun_out
VAR=SLIM_TRSV_CLUSTER VALS="4 8 16" CFG=2 REPS=1 bash tools/gpu_ab.sh > gpurun_out/ab1.log 2>&1
VAR=SLIM_BATCH VALS="8 16 24 32" CFG=2 REPS=1 bash tools/gpu_ab.sh >> gpurun_out/ab1.log 2>&1
cat gpurun_out/ab1.log
