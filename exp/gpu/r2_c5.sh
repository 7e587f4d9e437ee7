#!/bin/bash
# round 2: C5 (53-species, n = 54, global-norm mode) parity tests and a first bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "gri53" > gpurun_out/gpu_tests_c5.log 2>&1
tail -5 gpurun_out/gpu_tests_c5.log
timeout 1500 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 2500 gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err
