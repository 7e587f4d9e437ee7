#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/r_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/r_$tag.json 2>gpurun_out/r_$tag.err; }
run base
run l3 BDFB_LIB=exp/lib_l3.so
run l4 BDFB_LIB=exp/lib_l4.so
