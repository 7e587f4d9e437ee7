#!/bin/bash
# round-1 measurement: bench line + ncu launch list (same command) + full capture of the top kernel
mkdir -p gpurun_out
nproc > gpurun_out/host_nproc.txt; lscpu | head -20 > gpurun_out/host_lscpu.txt
python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
    python bench.py --no-cpu > gpurun_out/bench_r1_under_ncu.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:integrate -c 1 -o gpurun_out/prof_r1_full -f \
    python bench.py --steps 1 --warmup 0 --cells 262144 --no-cpu > gpurun_out/ncu_full_r1.log 2>&1
