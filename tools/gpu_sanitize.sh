#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize.py cases);
# logs under gpurun_out/sanitize/.  Usage: bash tools/gpu_sanitize.sh [cases...]
mkdir -p gpurun_out/sanitize
CASES=${@:-sim score snapshot cluster}
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize.py $c > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" | tee -a gpurun_out/sanitize/summary.txt
    tail -2 gpurun_out/sanitize/${tool}_${c}.log | tee -a gpurun_out/sanitize/summary.txt
  done
done
