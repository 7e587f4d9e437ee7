#!/bin/bash
# round 2: C5 (GRI-3.0-class n = 54, global-norm mode) launch list on a 262,144-cell slab
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python bench.py --config C5 --cells 262144 --steps 1 --warmup 0 --no-cpu > gpurun_out/c5_launches_bench.json 2> gpurun_out/c5_launches.err
tail -2 gpurun_out/c5_launches.err
timeout 900 python bench.py --config C5 --cells 262144 --steps 1 --warmup 1 --no-cpu > gpurun_out/c5_small_bench.json 2>&1
tail -c 400 gpurun_out/c5_small_bench.json
