#!/bin/bash
# round 2: ncu --set full of one mid-run K_ctl launch (C4 field, 1M cells) with source attribution
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:split_ctl_kernel -s 150 -c 1 -o gpurun_out/prof_ctl python bench.py --config C4 --cells 1048576 --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_ctl.log 2>&1
tail -2 gpurun_out/ncu_ctl.log
