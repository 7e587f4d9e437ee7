#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/t2_C4.json 2> gpurun_out/t2_C4.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t2_pytest.log 2>&1
echo "rc $?" >> gpurun_out/t2_pytest.log
