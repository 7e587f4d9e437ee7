#!/bin/bash
# round 2: racecheck / synccheck after the GROUP and THREAD fixes + their parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "thread or group" 2>&1 | tail -1
for tool in racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python exp/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run done" gpurun_out/sanitize_$tool.log | tail -3
done
