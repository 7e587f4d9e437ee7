#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tests/gpu_quick.py lu h2 drm > gpurun_out/j_quick.log 2>&1
timeout 900 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err
