#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sharded" > gpurun_out/pytest_rr.log 2>&1; echo "rr rc=$?" >> gpurun_out/pytest_rr.log
tail -4 gpurun_out/pytest_rr.log
timeout 900 python bench.py > gpurun_out/bench_cfg2_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg2_full.log
tail -2 gpurun_out/bench_cfg2_full.log | cut -c1-400
for c in 3 4; do
  timeout 900 python bench.py --config $c --quick --steps 16 > gpurun_out/bench_cfg${c}_quick.log 2>&1; echo "cfg$c rc=$?" >> gpurun_out/bench_cfg${c}_quick.log
  python -c "
import json,sys
for ln in open('gpurun_out/bench_cfg${c}_quick.log'):
    if ln.startswith('{'):
        d=json.loads(ln); print($c, d['value'], d['device_projector'], {k:(round(v['achieved_gbs']),round(v['frac'],3)) for k,v in d['streaming'].items() if isinstance(v,dict)})
"
  tail -1 gpurun_out/bench_cfg${c}_quick.log
done
CONFIGS="5" bash tools/gpu_stream.sh
