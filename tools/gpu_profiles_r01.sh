#!/bin/bash
# round-1 evidence refresh: full bench lines (all configs + reference arm),
# launch list of the headline config, ncu --set full of the streaming kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
for c in 2 1 3 4 5; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_full_cfg$c.log 2>&1; echo "cfg$c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CFG=2 bash tools/gpu_launches.sh
run_ncu() {  # name kernel-regex config skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $4 -c 1 \
    -o gpurun_out/ncu_$1 python bench.py --config $3 --steps 16 --warmup 3 --quick > gpurun_out/ncu_$1.log 2>&1
  echo "ncu $1 rc=$?"
}
run_ncu mtw_dense_cfg5 k_mtw_dense 5 40
run_ncu rowdot_cfg5 "k_rowdot<float, false" 5 40
run_ncu mtw_csc_cfg3 k_mtw_csc 3 20
run_ncu residual_csr_cfg3 k_residual_csr 3 20
run_ncu siddon_fill_cfg3 k_siddon_fill 3 0
