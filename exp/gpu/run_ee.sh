#!/bin/bash
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/ee_$tag.json 2>gpurun_out/ee_$tag.err; }
run base
run au4 BDFB_LIB=exp/lib_au4.so
