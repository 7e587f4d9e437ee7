#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"split_lu|split_jac" --launch-skip 400 -c 2 -o gpurun_out/i_lujac -f \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/i_lujac.log 2>&1
