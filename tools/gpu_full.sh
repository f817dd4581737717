#!/bin/bash
# full bench line + launch list + one full ncu capture of the batched Cholesky
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
CMD="python bench.py --steps 8 --warmup 3 --quick"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_chol_tiles -s 3 -c 1 -o gpurun_out/chol_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_csr -s 20 -c 1 -o gpurun_out/gram_full $CMD > gpurun_out/ncu_gram.log 2>&1
echo "gram rc=$?"
tail -2 gpurun_out/bench_full.log | cut -c1-300
