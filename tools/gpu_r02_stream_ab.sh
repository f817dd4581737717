#!/bin/bash
# streaming kernels, round-2 variants vs the previous ones: cold-L2 probe, iterate
# differences after 40 steps, then the full-run parity tests with the new Gram
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/stream_ab.log
: > $out
for cfg in 3 2 4; do
  SLIM_GRAM_LUT=1 SLIM_MTW_QUAD=6 timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep -E "config|rror" | sed "s/^/new /" >> $out
  SLIM_GRAM_LUT=0 timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep -E "config|rror" | sed "s/^/old /" >> $out
done
for cfg in 2 3 4; do
  SLIM_GRAM_LUT=1 SLIM_MTW_QUAD=6 timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_new_$cfg.npy
  SLIM_GRAM_LUT=0 SLIM_MTW_QUAD=6 timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_mid_$cfg.npy
  SLIM_GRAM_LUT=0 timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_old_$cfg.npy
  python -c "
import numpy as np
a=np.load('gpurun_out/x_new_$cfg.npy'); m=np.load('gpurun_out/x_mid_$cfg.npy'); b=np.load('gpurun_out/x_old_$cfg.npy')
print('config $cfg: mtw staged bit-identical:', np.array_equal(m,b), ' fixed-point Gram vs fp64 Gram rel diff:', float(np.linalg.norm(a-b)/np.linalg.norm(b)))" >> $out
done
rm -f gpurun_out/x_*.npy
cat $out
timeout 1500 python -m pytest tests/test_gpu_full_runs.py -m gpu -q -s > gpurun_out/full_runs_fx.log 2>&1
echo "rc=$?" >> gpurun_out/full_runs_fx.log
grep -E "error|passed|failed|rc=" gpurun_out/full_runs_fx.log | tail -20
