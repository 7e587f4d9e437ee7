#!/bin/bash
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/hh_$tag.json 2>gpurun_out/hh_$tag.err; }
run b16
run b64 BDFB_SPLIT_BATCH=64
run b4 BDFB_SPLIT_BATCH=4
