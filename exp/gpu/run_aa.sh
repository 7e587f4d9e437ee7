#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/aa_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/aa_$tag.json 2>gpurun_out/aa_$tag.err; }
run base
run k32 BDFB_LIB=exp/lib_k32.so
run k64 BDFB_LIB=exp/lib_k64.so
