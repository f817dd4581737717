#!/bin/bash
# configs[2]: factorization launch time alone vs in the pipeline, and the
# x-chain / Gram kernels' effect on it
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  echo "== $label" >> gpurun_out/contention.log
  env "$@" timeout 600 python tools/chol_order_sweep.py --config 3 --orders 1:32 --repeat 1 2>&1 | grep rep >> gpurun_out/contention.log
}
run default
run serial SLIM_SERIAL=1
run trsv8 SLIM_TRSV_CLUSTER=8
run trsv4 SLIM_TRSV_CLUSTER=4
run trsv1 SLIM_TRSV_CLUSTER=1
run xsms16 SLIM_XSMS=16
run xsms8 SLIM_XSMS=8
cat gpurun_out/contention.log
