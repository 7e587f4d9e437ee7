#!/bin/bash
# round-1 evidence for the final SPLIT kernels: default bench line, all configs, launch list (1M cells), ncu full
# captures of one mid-run launch of each split kernel (1M cells: K_ctl/K_rhs at launch 100, K_lu/K_jac at 100)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/f_C4.json 2> gpurun_out/f_C4.err
for c in C1 C2 C3 G4; do timeout 600 python bench.py --config $c > gpurun_out/f_$c.json 2> gpurun_out/f_$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
    python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/f_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"split_(ctl|rhs|lu|jac)" --launch-skip 400 -c 4 \
    -o gpurun_out/f_full -f python bench.py --no-cpu --steps 1 --warmup 0 --cells 1048576 > gpurun_out/f_full.log 2>&1
