#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:split_ctl --launch-skip 100 -c 1 -o gpurun_out/z_ctl -f \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/z_ctl.log 2>&1
