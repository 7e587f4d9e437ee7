#!/bin/bash
mkdir -p gpurun_out
export BDFB_SPLIT_SLOTS=65536 L=64 KS=split
ncu --set full --clock-control none --import-source on -k regex:split_ctl --launch-skip 400 -c 2 -o gpurun_out/e_ctl -f \
    python tests/gpu_quick.py time > gpurun_out/e_ctl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:split_rhs --launch-skip 200 -c 1 -o gpurun_out/e_rhs -f \
    python tests/gpu_quick.py time > gpurun_out/e_rhs.log 2>&1
