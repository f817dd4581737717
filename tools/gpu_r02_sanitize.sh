#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call: TOOL=memcheck|racecheck|synccheck|initcheck
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${TOOL:-memcheck}
for case in ${CASES:-dense tomo gen file}; do
  echo "== $T $case" >> gpurun_out/sanitize_$T.log
  timeout ${TLIM:-900} compute-sanitizer --tool $T --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_run.py $case >> gpurun_out/sanitize_$T.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$T.log
done
grep -E "==|rc=|ERROR SUMMARY|RACECHECK SUMMARY|ok|Error" gpurun_out/sanitize_$T.log | tail -30
