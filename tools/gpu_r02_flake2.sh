#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/shard_pytest.log
for i in $(seq 1 16); do
  timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sharded" 2>&1 | tail -n 1 >> gpurun_out/shard_pytest.log
done
sort gpurun_out/shard_pytest.log | cut -c1-30 | uniq -c
