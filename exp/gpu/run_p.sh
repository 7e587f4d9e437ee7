#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/p_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/p_$tag.json 2>gpurun_out/p_$tag.err; }
run base
run pf1 BDFB_LIB=exp/lib_pf1.so
run pf2 BDFB_LIB=exp/lib_pf2.so
