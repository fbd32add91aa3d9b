#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_driver.py: memcheck, racecheck, synccheck, initcheck
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_driver.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.txt
done
