#!/bin/bash
# C5 launch list (per-kernel device time) at a reduced cell count
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python bench.py --config C5 --cells 262144 --steps 1 --warmup 0 --no-cpu > gpurun_out/c5_launches_bench.log 2>&1
python exp/launch_summary.py gpurun_out/c5_launches.csv > gpurun_out/c5_launches_summary.txt 2>&1
cat gpurun_out/c5_launches_summary.txt | head -30
