#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/chol_trace.py 3982 > gpurun_out/trace.log 2>&1
timeout 300 python tools/chol_trace.py 600 >> gpurun_out/trace.log 2>&1
timeout 300 python tools/chol_trace.py 1086 >> gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
