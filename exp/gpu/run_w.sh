#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k full_size -v > gpurun_out/w_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:split_ctl --launch-skip 150 -c 1 -o gpurun_out/w_ctl -f \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 524288 > gpurun_out/w_ctl.log 2>&1
