#!/bin/bash
# ncu --set full of one full-window probe launch of the CSR Gram and M^T w kernels at configs[2]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export SLIM_MTW_QUAD=${SLIM_MTW_QUAD:-6}
ncu --set full --clock-control none --import-source on -k regex:k_gram_csr -s 12 -c 1 \
    -o gpurun_out/gram_fx_cfg3 -f python tools/stream_probe.py --config 3 --reps 4 > gpurun_out/ncu_gram_fx.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mtw_stage -s 2 -c 1 \
    -o gpurun_out/mtw_stage_cfg3 -f python tools/stream_probe.py --config 3 --reps 4 > gpurun_out/ncu_mtw_stage.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_residual_csr -s 12 -c 1 \
    -o gpurun_out/residual_cfg3 -f python tools/stream_probe.py --config 3 --reps 4 > gpurun_out/ncu_residual.log 2>&1
tail -n 3 gpurun_out/ncu_gram_fx.log; tail -n 3 gpurun_out/ncu_mtw_stage.log
