#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/u_pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/u_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1
echo "smoke rc $?" >> gpurun_out/u_smoke.log
