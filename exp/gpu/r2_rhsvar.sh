#!/bin/bash
# round 2: K_rhs organisation variants (instruction-cache locality) + block-synchronous ERK
mkdir -p gpurun_out
for v in 0 1 2; do
  BDFB_SPLIT_RHS_VAR=$v timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_rhsvar$v.json 2> gpurun_out/bench_c4_rhsvar$v.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_c4_rhsvar$v.json').read().splitlines()[-1]);print('var $v', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
done
timeout 900 python bench.py --config C4 --method erk4 --dt 1e-7 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_erk_sync.json 2> gpurun_out/bench_c4_erk_sync.err
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_erk_sync.json').read().splitlines()[-1]);print('erk', d['value'], d['roofline']['frac'])"
timeout 600 python -m pytest tests/test_gpu_solvers.py -q -p no:cacheprovider -k erk 2>&1 | tail -2
