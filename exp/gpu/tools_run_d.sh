#!/bin/bash
mkdir -p gpurun_out
export BDFB_SPLIT_SLOTS=65536 L=64 KS=split
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_launches.csv \
    python tests/gpu_quick.py time > gpurun_out/d_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:split_ctl --launch-skip 40 -c 1 -o gpurun_out/d_ctl -f \
    python tests/gpu_quick.py time > gpurun_out/d_ctl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:split_rhs --launch-skip 40 -c 1 -o gpurun_out/d_rhs -f \
    python tests/gpu_quick.py time > gpurun_out/d_rhs.log 2>&1
