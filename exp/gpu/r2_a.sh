#!/bin/bash
# round 2: transcendental weights (ncu on the probe), new GPU tests, default bench line
set -x
mkdir -p gpurun_out
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
timeout 300 ncu --metrics $M --csv exp/probe/transc_probe > gpurun_out/transc_probe_ncu.csv 2> gpurun_out/transc_probe_ncu.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "nccl or split_lu or global_norm" > gpurun_out/gpu_tests_r2b.log 2>&1
tail -3 gpurun_out/gpu_tests_r2b.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
tail -c 3000 gpurun_out/bench_r2a.json
