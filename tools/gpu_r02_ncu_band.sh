#!/bin/bash
# does the banded ticket order cut k_chol_i8's DRAM traffic (configs[2])? and a 4-stage ring
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_1912_07962_b200
for v in default nst4; do
  if [ $v = nst4 ]; then export SLIM_LIB=$L/libslimb200_nst4.so; else unset SLIM_LIB; fi
  for s in 0 1; do
    echo "== $v serial=$s" >> gpurun_out/band_nst.log
    SLIM_SERIAL=$([ $s = 1 ] && echo 1) timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32,4:32 --repeat 1 2>&1 | grep rep >> gpurun_out/band_nst.log
  done
done
unset SLIM_LIB
CMD="python bench.py --config 3 --steps 16 --warmup 3 --bare"
SLIM_CHOL_COLS=4 $CMD > gpurun_out/ncu_plain_band.log 2>&1 &&
SLIM_CHOL_COLS=4 ncu --set full --clock-control none -k regex:k_chol_i8 -s 8 -c 1 \
    -o gpurun_out/chol_cfg3_band4 $CMD > gpurun_out/ncu_band.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_band.log
cat gpurun_out/band_nst.log; tail -2 gpurun_out/ncu_band.log
