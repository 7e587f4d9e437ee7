#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "autoignition" -s > gpurun_out/ai_pytest.log 2>&1
echo "rc $?" >> gpurun_out/ai_pytest.log
