#!/bin/bash
# split-kernel: parity vs oracle (small), timing at 64^3, launch list, full-size bench
mkdir -p gpurun_out
rm -f gpurun_out/c_time.log
timeout 600 python tests/gpu_quick.py h2 drm > gpurun_out/c_quick.log 2>&1
for S in 65536 262144; do
  BDFB_SPLIT_SLOTS=$S L=64 KS=split timeout 300 python tests/gpu_quick.py time >> gpurun_out/c_time.log 2>&1
done
BDFB_SPLIT_SLOTS=65536 L=64 KS=split ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches.csv \
    python tests/gpu_quick.py time > gpurun_out/c_l.log 2>&1
for S in 262144 1048576; do
BDFB_SPLIT_SLOTS=$S timeout 600 python bench.py --kernel split --no-cpu --steps 2 --warmup 1 > gpurun_out/c_bench_split_$S.json 2> gpurun_out/c_bench_split.err
done
