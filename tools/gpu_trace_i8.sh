mkdir -p gpurun_out
SLIM_CHOL_TRACE=gpurun_out/trace_cfg${CFG:-2}.csv SLIM_CHOL_TRACE_LAUNCH=${TL:-4} timeout 600 python bench.py --config ${CFG:-2} --quick --steps 32 > gpurun_out/trace_bench.log 2>&1
python tools/trace_phases.py gpurun_out/trace_cfg${CFG:-2}.csv
