#!/bin/bash
# round 2: compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small problems)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python exp/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run done" gpurun_out/sanitize_$tool.log | tail -3
done
