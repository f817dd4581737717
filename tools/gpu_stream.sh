#!/bin/bash
# streaming-kernel probe (bench "streaming") on every configuration, quick bench lines
mkdir -p gpurun_out
for c in ${CONFIGS:-2 1 3 4 5}; do
  timeout 900 python bench.py --config $c --quick --steps ${STEPS:-32} > gpurun_out/stream_cfg$c.log 2>&1; echo "cfg$c rc=$?" >> gpurun_out/stream_cfg$c.log
  python - "$c" << 'PY'
import json, sys
c = sys.argv[1]
lines = open(f"gpurun_out/stream_cfg{c}.log").read().splitlines()
for ln in lines:
    if ln.startswith("{"):
        d = json.loads(ln)
        st = {k: (round(v["us_per_launch"], 1), round(v["bytes_per_launch"] / 1e6, 2), round(v["achieved_gbs"]), round(v["frac"], 3))
              for k, v in d["streaming"].items() if isinstance(v, dict)}
        print(c, round(d["value"], 2), "it/s", st)
        break
else:
    print(c, "FAILED", lines[-5:])
PY
done
