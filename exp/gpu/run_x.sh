#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/x_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run base
run b2 BDFB_SPLIT_CTL_SMEM=100000
run b1 BDFB_SPLIT_CTL_SMEM=110000
