#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/g_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
