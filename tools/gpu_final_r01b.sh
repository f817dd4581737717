#!/bin/bash
# round-1 evidence after the 8-bit trailing digits (SLIM_QD=7 SLIM_DBITS=8):
# (build the comparison library first, in the build container:
#  SLIM_NVCC_EXTRA="-DSLIM_QD=8 -DSLIM_DBITS=7" python -m paper_1912_07962_b200.build &&
#  mv paper_1912_07962_b200/libslimb200.so paper_1912_07962_b200/libslimb200_d7.so &&
#  python -m paper_1912_07962_b200.build)
# factorization accuracy vs the previous layout (libslimb200_d7.so), GPU suite,
# smoke, full bench lines, reference arm, launch list, ncu of k_chol_i8
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python tools/chol_check.py 3982 8000 13032 > gpurun_out/chol_check_d8.log 2>&1
SLIM_LIB=$PWD/paper_1912_07962_b200/libslimb200_d7.so timeout 300 python tools/chol_check.py 3982 8000 13032 > gpurun_out/chol_check_d7.log 2>&1
cat gpurun_out/chol_check_d8.log gpurun_out/chol_check_d7.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 1 3 4 5; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_full_cfg$c.log 2>&1; echo "cfg$c rc=$?"; tail -1 gpurun_out/bench_full_cfg$c.log | cut -c1-200
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CFG=2 bash tools/gpu_launches.sh
for c in 2 3; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_chol_i8 -s 2 -c 1 \
    -o gpurun_out/chol_full_cfg$c python bench.py --steps 32 --warmup 3 --bare --config $c > gpurun_out/ncu_full_cfg$c.log 2>&1
  echo "ncu cfg$c rc=$?"
done
