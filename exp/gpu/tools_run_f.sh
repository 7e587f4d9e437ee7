#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/f_time.log
BDFB_SPLIT_SLOTS=65536 L=64 KS=split timeout 300 python tests/gpu_quick.py time >> gpurun_out/f_time.log 2>&1
BDFB_SPLIT_SLOTS=65536 L=64 KS=split ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
    python tests/gpu_quick.py time > gpurun_out/f_l.log 2>&1
BDFB_SPLIT_SLOTS=65536 L=64 KS=split ncu --set full --clock-control none --import-source on -k regex:split_ctl --launch-skip 300 -c 1 -o gpurun_out/f_ctl -f \
    python tests/gpu_quick.py time > gpurun_out/f_ctl.log 2>&1
BDFB_SPLIT_SLOTS=262144 timeout 600 python bench.py --kernel split --no-cpu --steps 2 --warmup 1 > gpurun_out/f_bench_split.json 2> gpurun_out/f_bench_split.err
