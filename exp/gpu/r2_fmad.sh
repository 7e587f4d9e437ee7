#!/bin/bash
# round 2: contraction in the RHS translation unit (rhs.cu) + out-of-line ERK RHS: parity + benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solvers.py -q -p no:cacheprovider -x > gpurun_out/gpu_fmad.log 2>&1
tail -3 gpurun_out/gpu_fmad.log
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "== $name rc=$?"; tail -3 gpurun_out/bench_$name.err; }
run c4_fmad --config C4 --steps 3 --warmup 3 --no-cpu
run c4_erk_dt1e-7_b --config C4 --method erk4 --dt 1e-7 --steps 3 --warmup 3 --no-cpu
