#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/dq_pytest.log 2>&1
echo "rc $?" >> gpurun_out/dq_pytest.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "dq" -s > gpurun_out/dq_pytest_s.log 2>&1
timeout 900 python bench.py --no-cpu --jac dq --steps 2 --warmup 1 > gpurun_out/dq_bench.json 2> gpurun_out/dq_bench.err
