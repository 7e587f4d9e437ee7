#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "flame_parity or edge or sharding or full_size_c3" > gpurun_out/gg_pytest.log 2>&1
echo "rc $?" >> gpurun_out/gg_pytest.log
BDFB_SPLIT_OVERLAP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "flame_parity or sharding" > gpurun_out/gg_pytest_ovl.log 2>&1
echo "rc $?" >> gpurun_out/gg_pytest_ovl.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/gg_$tag.json 2>gpurun_out/gg_$tag.err; }
run base
run ovl BDFB_SPLIT_OVERLAP=1
