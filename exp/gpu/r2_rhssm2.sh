#!/bin/bash
# round 2: shared-memory e^{-g/RT} RHS as default (K_rhs VAR 3; erk_eval; eval diagnostic): parity + benches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_rhssm.log 2>&1; tail -1 gpurun_out/gpu_rhssm.log
for v in 3 4; do
  BDFB_SPLIT_RHS_VAR=$v timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_rhs$v.json 2> gpurun_out/bench_c4_rhs$v.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_c4_rhs$v.json').read().splitlines()[-1]);print('var $v', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()}, d['phases']['rhs']['frac'])"
done
timeout 900 python bench.py --config C4 --method erk4 --dt 1e-7 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_erk_sm.json 2> gpurun_out/bench_erk_sm.err
python -c "import json;d=json.loads(open('gpurun_out/bench_erk_sm.json').read().splitlines()[-1]);print('erk', d['value'], d['roofline']['frac'])"
