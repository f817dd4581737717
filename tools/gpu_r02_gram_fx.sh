#!/bin/bash
# fixed-point CSR Gram (default) vs fp64 k_gram_csr (SLIM_GRAM_LUT=0): probe, iterate difference, ncu
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/gram_fx_ab.log
: > $out
for cfg in 3 2 4; do
  SLIM_GRAM_LUT=1 timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep -E "gram|rror" | sed "s/^/fx   /" >> $out
  SLIM_GRAM_LUT=0 timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep -E "gram|rror" | sed "s/^/fp64 /" >> $out
done
for cfg in 2 3 4; do
  SLIM_GRAM_LUT=1 timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_new_$cfg.npy
  SLIM_GRAM_LUT=0 timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_old_$cfg.npy
  python -c "
import numpy as np
a=np.load('gpurun_out/x_new_$cfg.npy'); b=np.load('gpurun_out/x_old_$cfg.npy')
print('config $cfg: fixed-point Gram vs fp64 Gram, relative iterate difference after 40 steps:', float(np.linalg.norm(a-b)/np.linalg.norm(b)))" >> $out
done
rm -f gpurun_out/x_*.npy
cat $out
ncu --set full --clock-control none --import-source on -k regex:k_gram_csr -s 12 -c 1 \
    -o gpurun_out/gram_fx_cfg3 -f python tools/stream_probe.py --config 3 --reps 4 > gpurun_out/ncu_gram_fx.log 2>&1
