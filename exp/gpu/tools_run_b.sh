#!/bin/bash
# ncu evidence for the thread-per-cell C4 kernel: launch list of the bench command + full capture at 262144 cells
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches_c4.csv \
    python bench.py --steps 1 --warmup 1 --cells 1048576 --no-cpu > gpurun_out/b_bench_under_ncu.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:integrate -c 1 -o gpurun_out/b_prof_tpc_c4 -f \
    python bench.py --steps 1 --warmup 0 --cells 262144 --no-cpu > gpurun_out/b_ncu_full.log 2>&1
