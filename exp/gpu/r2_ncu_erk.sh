#!/bin/bash
# round 2: ncu --set full on the ERK kernel (C4 cells at dt 1e-7)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:erk_kernel -s 1 -c 1 -o gpurun_out/prof_erk python bench.py --config C4 --method erk4 --dt 1e-7 --cells 262144 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_erk.log 2>&1
tail -3 gpurun_out/ncu_erk.log
