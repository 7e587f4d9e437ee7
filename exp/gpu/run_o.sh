#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/o_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 2097152 > gpurun_out/o_$tag.json 2>/dev/null; }
run s16k BDFB_SPLIT_SLOTS=16384 BDFB_SPLIT_BATCH=64
run s32k BDFB_SPLIT_SLOTS=32768 BDFB_SPLIT_BATCH=64
run s65k BDFB_SPLIT_SLOTS=65536 BDFB_SPLIT_BATCH=32
