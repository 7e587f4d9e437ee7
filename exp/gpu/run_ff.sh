#!/bin/bash
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/ff_$tag.json 2>gpurun_out/ff_$tag.err; }
run base
run est BDFB_LIB=exp/lib_est.so
BDFB_LIB=exp/lib_est.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity or flame_parity" > gpurun_out/ff_pytest.log 2>&1
echo "rc $?" >> gpurun_out/ff_pytest.log
