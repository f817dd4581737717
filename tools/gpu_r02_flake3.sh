#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/shard_stress4.log
run() {  # label, P, env...
  label=$1; P=$2; shift; shift
  for rep in 1 2 3 4; do
    echo "== $label (process $rep)" >> gpurun_out/shard_stress4.log
    env "$@" timeout 200 python tools/shard_stress.py 400 $P 2>&1 | grep -v "^  " | grep -v "PriorityRange" | head -3 | cut -c1-250 >> gpurun_out/shard_stress4.log
  done
}
run "P=3, legacy-stream copies awaited, no group sync" 3 X=1
run "P=4, legacy-stream copies awaited, no group sync" 4 X=1
cat gpurun_out/shard_stress4.log
