#!/bin/bash
mkdir -p gpurun_out
for c in ${CONFIGS:-1 3 4 5}; do
  timeout 900 python bench.py --config $c --quick --steps ${STEPS:-32} > gpurun_out/bench_cfg$c.log 2>&1; echo "cfg$c rc=$?" >> gpurun_out/bench_cfg$c.log
  python - "$c" << 'PY'
import json, sys
c = sys.argv[1]
lines = open(f"gpurun_out/bench_cfg{c}.log").read().splitlines()
for ln in lines:
    if ln.startswith("{"):
        d = json.loads(ln)
        print(c, round(d["value"], 2), "it/s", round(d["rows_per_s"]), "rows/s frac", round(d["roofline"]["frac"], 3),
              "agg", round(d["roofline"]["aggregate_frac"], 3), d["kernel_ms_per_step"], d["roofline"]["launches"])
        break
else:
    print(c, "FAILED", lines[-5:])
PY
done
