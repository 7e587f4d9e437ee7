#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gl_lu -s 1 -c 1 -o gpurun_out/prof_glu python bench.py --config C5 --cells 65536 --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_glu.log 2>&1
tail -2 gpurun_out/ncu_glu.log
