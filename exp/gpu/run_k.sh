#!/bin/bash
# K_ctl variants (TS staging / occupancy) and slot-pool sizes on 1M cells of the C4 field
mkdir -p gpurun_out
rm -f gpurun_out/k_*.json
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 --cells 1048576 > gpurun_out/k_$tag.json 2>/dev/null; }
run base
run g3 BDFB_LIB=exp/lib_g3.so
run g4 BDFB_LIB=exp/lib_g4.so
run g5 BDFB_LIB=exp/lib_g5.so
run s131k BDFB_SPLIT_SLOTS=131072
run s524k BDFB_SPLIT_SLOTS=524288
run g4s524k BDFB_LIB=exp/lib_g4.so BDFB_SPLIT_SLOTS=524288
