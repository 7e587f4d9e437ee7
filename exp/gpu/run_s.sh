#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/s_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/s_$tag.json 2>gpurun_out/s_$tag.err; }
run base1
run l3 BDFB_LIB=exp/lib_l3.so
run base2
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/s_smi.txt
