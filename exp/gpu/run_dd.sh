#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity or jacobian_parity or flame_parity or full_size_c3" > gpurun_out/dd_pytest.log 2>&1
echo "rc $?" >> gpurun_out/dd_pytest.log
timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/dd_sel.json 2>gpurun_out/dd_sel.err
