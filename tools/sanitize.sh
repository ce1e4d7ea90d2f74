#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py: memcheck, racecheck, synccheck, initcheck.
# Summaries go to gpurun_out/sanitize_<tool>.log (copied to profiles/ by hand).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  tail -4 gpurun_out/sanitize_$tool.log
done
