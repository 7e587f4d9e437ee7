#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "flame_parity or sharding or full_size_c3" > gpurun_out/ii_pytest.log 2>&1
echo "rc $?" >> gpurun_out/ii_pytest.log
timeout 600 python tests/gpu_quick.py drm > gpurun_out/ii_quick.log 2>&1
timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/ii_diag.json 2>gpurun_out/ii_diag.err
