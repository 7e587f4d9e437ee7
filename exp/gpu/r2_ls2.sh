#!/bin/bash
# round 2: solver tests (GMRES / CVDiag / ERK) without -x, failure lines only
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_solvers.py -q -s -p no:cacheprovider > gpurun_out/gpu_solvers.log 2>&1
grep -E "identical|AssertionError|passed|failed|Error" gpurun_out/gpu_solvers.log | head -60
