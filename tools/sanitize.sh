#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (tools/sanitize_cases.py); summaries land in gpurun_out/sanitize_*.log.
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE_CASES_OK|Error|error" gpurun_out/sanitize_$tool.log | tail -5
done
