#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/y_*.json
timeout 600 python tests/gpu_quick.py h2 drm > gpurun_out/y_quick.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "flame_parity or edge or sharding or typical" > gpurun_out/y_pytest.log 2>&1
echo "rc $?" >> gpurun_out/y_pytest.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/y_$tag.json 2>gpurun_out/y_$tag.err; }
run base
