#!/bin/bash
# CSR Gram with prefetched batches (libslimb200_gpf.so) vs default: cold-L2 probe and bits
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_1912_07962_b200
for cfg in 3 2 4; do
  for v in default gpf; do
    if [ $v = default ]; then unset SLIM_LIB; else export SLIM_LIB=$L/libslimb200_$v.so; fi
    timeout 300 python tools/stream_probe.py --config $cfg 2>&1 | grep gram | sed "s/^/$v /" >> gpurun_out/gram_ab.log
  done
done
for cfg in 2 3; do
  unset SLIM_LIB; timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_def_$cfg.npy
  SLIM_LIB=$L/libslimb200_gpf.so timeout 300 python tools/bits_run.py $cfg 40 gpurun_out/x_gpf_$cfg.npy
  python -c "import numpy as np; a=np.load('gpurun_out/x_def_$cfg.npy'); b=np.load('gpurun_out/x_gpf_$cfg.npy'); print('config $cfg bit-identical:', np.array_equal(a,b))" >> gpurun_out/gram_ab.log
done
rm -f gpurun_out/x_*.npy
cat gpurun_out/gram_ab.log
