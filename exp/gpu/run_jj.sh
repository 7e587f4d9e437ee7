#!/bin/bash
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/jj_$tag.json 2>gpurun_out/jj_$tag.err; }
run base
run full BDFB_SPLIT_RHS_FULLGRID=1
