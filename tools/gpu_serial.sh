# uncontended kernel times: factorization and x-chain serialised (debug knob)
mkdir -p gpurun_out
VAR=SLIM_SERIAL VALS="1" CFG=${CFG:-2} REPS=1 bash tools/gpu_ab.sh > gpurun_out/serial.log 2>&1
for c in 1 3 4 5; do VAR=SLIM_SERIAL VALS="1" CFG=$c REPS=1 STEPS=32 bash tools/gpu_ab.sh >> gpurun_out/serial.log 2>&1; done
cat gpurun_out/serial.log
