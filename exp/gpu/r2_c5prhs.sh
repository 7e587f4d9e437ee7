#!/bin/bash
# round 2: C5P K_rhs with the shared-memory RHS (VAR 3, 108 KB per 128-thread block) vs registers (VAR 0)
mkdir -p gpurun_out
for v in 0 3; do
  BDFB_SPLIT_RHS_VAR=$v timeout 900 python bench.py --config C5P --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c5p_rhs$v.json 2> gpurun_out/bench_c5p_rhs$v.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_c5p_rhs$v.json').read().splitlines()[-1]);print('var $v', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
done
