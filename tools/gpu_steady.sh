# steady-state vs default window; overlapped numbers for the other configs
mkdir -p gpurun_out
VAR=SLIM_X VALS="0" CFG=2 REPS=1 STEPS=480 bash tools/gpu_ab.sh > gpurun_out/steady.log 2>&1
for c in 3 4 5; do VAR=SLIM_X VALS="0" CFG=$c REPS=1 STEPS=32 bash tools/gpu_ab.sh >> gpurun_out/steady.log 2>&1; done
cat gpurun_out/steady.log
