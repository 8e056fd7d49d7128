#!/bin/bash
# compute-sanitizer over profiles/sanitize_cases.py; logs to gpurun_out/sanitizer_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python profiles/sanitize_cases.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_summary.txt
done
cat gpurun_out/sanitizer_summary.txt
