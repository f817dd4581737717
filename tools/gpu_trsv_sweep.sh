#!/bin/bash
# triangular-solve cluster size sweep on one configuration + isolated launch list
set -u
mkdir -p gpurun_out
for C in ${CS:-4 8 16}; do
  SLIM_TRSV_CLUSTER=$C timeout 600 python bench.py --config ${CFG:-2} --quick --steps 32 > gpurun_out/sweep_C$C.log 2>&1
  python - "$C" << 'PY'
import json, sys
C = sys.argv[1]
ln = [l for l in open(f"gpurun_out/sweep_C{C}.log") if l.startswith("{")]
if ln:
    d = json.loads(ln[-1]); print("C", C, round(d["value"], 1), "it/s", d["kernel_ms_per_step"])
else:
    print("C", C, "FAILED", open(f"gpurun_out/sweep_C{C}.log").read()[-400:])
PY
done
CFG=${CFG:-2} STEPS=16 bash tools/gpu_launches.sh > /dev/null 2>&1; echo "launches rc=$?"
