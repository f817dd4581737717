# int8 tensor-core factorization vs DMMA: standalone potrf accuracy/time, then quick bench
mkdir -p gpurun_out
(SLIM_CHOL=dmma timeout 300 python tools/chol_check.py ${NS:-100 600 1000 3982 8000}; \
 SLIM_CHOL=i8 timeout 300 compute-sanitizer --tool memcheck python tools/chol_check.py 200 2>&1 | tail -5; \
 SLIM_CHOL=i8 timeout 300 python tools/chol_check.py ${NS:-100 600 1000 3982 8000}) > gpurun_out/i8.log 2>&1
echo "rc=$?" >> gpurun_out/i8.log
cat gpurun_out/i8.log
