#!/bin/bash
# round 2: ERK block size (resident threads per SM vs the L2-resident workspace)
mkdir -p gpurun_out
for v in 256 192; do
  BDFB_LIB=exp/lib_erk$v.so timeout 900 python bench.py --config C4 --method erk4 --dt 1e-7 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_erk$v.json 2> gpurun_out/bench_erk$v.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_erk$v.json').read().splitlines()[-1]);print('erk $v', d['value'], d['roofline']['frac'])"
done
