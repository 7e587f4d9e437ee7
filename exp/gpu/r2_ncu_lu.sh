#!/bin/bash
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:split_lu_kernel -s 150 -c 1 -o gpurun_out/prof_lu python bench.py --config C4 --cells 1048576 --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_lu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:split_jac_kernel -s 150 -c 1 -o gpurun_out/prof_jac python bench.py --config C4 --cells 1048576 --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_jac.log 2>&1
tail -1 gpurun_out/ncu_lu.log gpurun_out/ncu_jac.log
