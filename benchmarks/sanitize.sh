#!/bin/bash
# compute-sanitizer over benchmarks/sanitize.py, kernels of the qnmt namespace only.
# Logs: gpurun_out/sanitize_{memcheck,racecheck,synccheck}.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-regex kns=qnmt --print-limit 50 \
    python benchmarks/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
