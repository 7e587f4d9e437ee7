#!/bin/bash
# round 2: bulk L2 prefetch of the warp's Nordsieck (3) / state (4) rows at the start of K_ctl
mkdir -p gpurun_out
for v in pf3 pf4; do
  BDFB_LIB=exp/lib_$v.so timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_$v.json 2> gpurun_out/bench_c4_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_c4_$v.json').read().splitlines()[-1]);print('$v', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
done
