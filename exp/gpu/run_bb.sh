#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/bb_*.json
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/bb_$tag.json 2>gpurun_out/bb_$tag.err; }
run s524k BDFB_SPLIT_SLOTS=524288
run s786k BDFB_SPLIT_SLOTS=786432
run s1m BDFB_SPLIT_SLOTS=1048576
