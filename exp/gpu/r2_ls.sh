#!/bin/bash
# round 2: matrix-free linear solvers (CVDiag, GMRES) parity + the full GPU suite after the SPLIT refactor
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py -x -q -s -p no:cacheprovider > gpurun_out/gpu_solvers.log 2>&1
tail -30 gpurun_out/gpu_solvers.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_solvers.py > gpurun_out/gpu_all.log 2>&1
tail -5 gpurun_out/gpu_all.log
