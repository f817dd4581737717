#!/bin/bash
# CSR Gram through per-column records (k_gram_lut + k_gram_csr_lut, default) vs the
# pointer-chasing k_gram_csr (SLIM_GRAM_LUT=0): cold-L2 probe and bit-for-bit iterates
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/gram_lut_ab.log
: > $out
for cfg in 3 2 4; do
  for v in 1 0; do
    SLIM_GRAM_LUT=$v timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep -E "gram|Error|error" | sed "s/^/lut=$v /" >> $out
  done
done
for cfg in 2 3 4; do
  SLIM_GRAM_LUT=1 timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_lut_$cfg.npy
  SLIM_GRAM_LUT=0 timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_old_$cfg.npy
  python -c "import numpy as np; a=np.load('gpurun_out/x_lut_$cfg.npy'); b=np.load('gpurun_out/x_old_$cfg.npy'); print('config $cfg bit-identical:', np.array_equal(a,b), float(np.abs(a-b).max()))" >> $out
done
rm -f gpurun_out/x_*.npy
cat $out
