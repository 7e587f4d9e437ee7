#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/q_*.json
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "flame_parity or edge or sharding or robertson or full_size_c3" > gpurun_out/q_pytest.log 2>&1
echo "rc $?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/q_base.json 2>gpurun_out/q_base.err
