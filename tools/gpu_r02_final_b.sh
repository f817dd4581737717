#!/bin/bash
# round-2 final: the whole -m gpu suite, smoke, the reference arm, then the bench lines of every configuration
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -rA > gpurun_out/final_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/final_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_ref.out 2> gpurun_out/final_ref.err
echo "ref rc=$?" >> gpurun_out/final_ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench.out 2> gpurun_out/final_bench.err
echo "bench rc=$?" >> gpurun_out/final_bench.err
for cfg in 1 2 4 5; do
  st=20; [ $cfg = 2 ] && st=176; [ $cfg = 1 ] && st=176; [ $cfg = 5 ] && st=160
  timeout 900 python bench.py --config $cfg --gpus 1 --steps $st --warmup 5 > gpurun_out/final_bench_cfg$cfg.out 2> gpurun_out/final_bench_cfg$cfg.err
  echo "bench cfg$cfg rc=$?" >> gpurun_out/final_bench_cfg$cfg.err
done
tail -n 2 gpurun_out/final_suite.log | cut -c1-120; tail -n 1 gpurun_out/final_smoke.log gpurun_out/final_ref.err gpurun_out/final_bench.err gpurun_out/final_bench_cfg*.err
