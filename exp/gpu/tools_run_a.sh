#!/bin/bash
mkdir -p gpurun_out
nvidia-smi > gpurun_out/a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/a_pytest_gpu.log
L=64 timeout 600 python tests/gpu_quick.py time > gpurun_out/a_time64.log 2>&1
timeout 900 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
