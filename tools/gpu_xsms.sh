# SM partition A/B: x-chain on its own green context of SLIM_XSMS SMs
mkdir -p gpurun_out
: > gpurun_out/xsms.log
for c in ${CFGS:-2 3 1 5}; do VAR=SLIM_XSMS VALS="${VALS:-0 16 24}" CFG=$c REPS=1 STEPS=${STEPS:-48} bash tools/gpu_ab.sh >> gpurun_out/xsms.log 2>&1; done
cat gpurun_out/xsms.log
