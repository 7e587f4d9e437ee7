#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tests/gpu_quick.py h2 drm > gpurun_out/cc_quick.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "flame_parity or edge or sharding or typical or full_size_c3" > gpurun_out/cc_pytest.log 2>&1
echo "rc $?" >> gpurun_out/cc_pytest.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/cc_$tag.json 2>gpurun_out/cc_$tag.err; }
run init
run noinit BDFB_LIB=exp/lib_noinit.so
run ik4 BDFB_LIB=exp/lib_ik4.so
