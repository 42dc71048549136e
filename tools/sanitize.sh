#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_workload.py
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error" gpurun_out/sanitize_$tool.log | tail -3
done
