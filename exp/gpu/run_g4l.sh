#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g4_launches.csv \
    python bench.py --config G4 --no-cpu --steps 1 --warmup 0 > gpurun_out/g4_l.log 2>&1
