#!/bin/bash
# compute-sanitizer over small launches of every kernel family; logs -> gpurun_out/sanitizer/
mkdir -p gpurun_out/sanitizer
python tools/sanitize_cases.py > gpurun_out/sanitizer/plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitizer/plain.log; exit 1; }
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all cases ok" gpurun_out/sanitizer/$tool.log | tail -3
done
