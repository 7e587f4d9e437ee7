#!/bin/bash
# bench lines of every config with the current kernels
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/t_C4.json 2> gpurun_out/t_C4.err
for c in C1 C2 C3 G4; do timeout 600 python bench.py --config $c > gpurun_out/t_$c.json 2> gpurun_out/t_$c.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/t_ref.json 2> gpurun_out/t_ref.err
