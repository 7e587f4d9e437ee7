#!/bin/bash
# usage: tools_profile.sh <tag> <config> <cells>
tag=$1; cfg=${2:-C4}; cells=${3:-65536}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --config $cfg --steps 1 --warmup 0 --cells $cells --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:integrate -c 1 -o gpurun_out/prof_${tag} -f \
    python bench.py --config $cfg --steps 1 --warmup 0 --cells $cells --no-cpu > gpurun_out/ncu_${tag}.log 2>&1
