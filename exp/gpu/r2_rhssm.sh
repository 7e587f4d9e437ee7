#!/bin/bash
# round 2: generated RHS with cv first (y dies early) and the shared-memory e^{-g/RT} variant (VAR 3)
mkdir -p gpurun_out
for v in 0 3; do
  BDFB_SPLIT_RHS_VAR=$v timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_rhs$v.json 2> gpurun_out/bench_c4_rhs$v.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_c4_rhs$v.json').read().splitlines()[-1]);print('var $v', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()}, d['phases']['rhs']['frac'])"
done
BDFB_SPLIT_RHS_VAR=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "flame_parity and split" 2>&1 | tail -1
