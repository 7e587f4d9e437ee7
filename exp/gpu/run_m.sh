#!/bin/bash
# round-1 evidence for the SPLIT design: default bench line (with cpu_baseline), ncu launch list of the bench
# command on 1M cells, one ncu --set full capture of each split kernel mid-run (262144 cells)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches.csv \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/m_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"split_(ctl|rhs|lu|jac)" --launch-skip 600 -c 4 \
    -o gpurun_out/m_full -f python bench.py --no-cpu --steps 1 --warmup 0 --cells 262144 > gpurun_out/m_full.log 2>&1
