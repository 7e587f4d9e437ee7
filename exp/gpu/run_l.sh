#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/l_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/l_$tag.json 2>/dev/null; }
run base
run m2 BDFB_LIB=exp/lib_m2.so
run b64 BDFB_LIB=exp/lib_b64.so
run b256 BDFB_LIB=exp/lib_b256.so
