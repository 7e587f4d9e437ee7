#!/bin/bash
# bench (split default) + ncu launch list of the same command at 1M cells + full captures of K_ctl and K_rhs
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_launches.csv \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/h_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:split_ctl --launch-skip 100 -c 1 -o gpurun_out/h_ctl -f \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/h_ctl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:split_rhs --launch-skip 100 -c 1 -o gpurun_out/h_rhs -f \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/h_rhs.log 2>&1
