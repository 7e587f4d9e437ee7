#!/bin/bash
# round 2: bench lines of the new rows on C4 (256^3 DRM19-class): GMRES (1A), CVDiag, ERK vs BDF at dt 1e-7
mkdir -p gpurun_out
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "== $name rc=$?"; tail -c 600 gpurun_out/bench_$name.json; echo; tail -3 gpurun_out/bench_$name.err; }
run c4_gmres --config C4 --ls gmres --steps 3 --warmup 3
run c4_erk_dt1e-7 --config C4 --method erk4 --dt 1e-7 --steps 3 --warmup 3
run c4_bdf_dt1e-7 --config C4 --dt 1e-7 --steps 3 --warmup 3 --no-cpu
run c4_gmres_dt1e-7 --config C4 --ls gmres --dt 1e-7 --steps 3 --warmup 3 --no-cpu
run c4_diag --config C4 --ls diag --steps 2 --warmup 1 --no-cpu
