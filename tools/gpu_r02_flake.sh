#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/shard_stress.log
run() {  # label, env...
  label=$1; shift
  for rep in 1 2 3; do
    echo "== $label (process $rep)" >> gpurun_out/shard_stress.log
    env "$@" timeout 150 python tools/shard_stress.py ${REPS:-400} ${P:-3} 2>&1 | grep -v "^  " | grep -v "PriorityRange" | head -3 | cut -c1-250 >> gpurun_out/shard_stress.log
  done
}
P=3 run "P=3, groups of three or more synchronise at every exchange" X=1
P=4 run "P=4, groups of three or more synchronise at every exchange" X=1
cat gpurun_out/shard_stress.log
