#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "global" > gpurun_out/g4_pytest.log 2>&1
echo "rc $?" >> gpurun_out/g4_pytest.log
timeout 1200 python bench.py --config G4 > gpurun_out/g4_128.json 2> gpurun_out/g4_128.err
