#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/n_*.json
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rhs_parity or jacobian_parity or flame_parity" > gpurun_out/n_pytest.log 2>&1
echo "rc $?" >> gpurun_out/n_pytest.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/n_$tag.json 2>/dev/null; }
run base
run pf BDFB_LIB=exp/lib_pf.so
