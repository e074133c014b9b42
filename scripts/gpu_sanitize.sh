#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small inputs on every plan
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export TCUDB_CALIBRATE=0   # keep the sanitized runs small (the calibration is covered by the GPU tests)
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout -s KILL 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python scripts/sanitize_cases.py quick > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|SANITIZE_CASES_OK|RACECHECK SUMMARY" gpurun_out/sanitize_$tool.log | tail -3
done
