#!/bin/bash
# round 2: thread-per-entry generated Jacobian (jac_cm) for K_jac vs the group Jacobian
mkdir -p gpurun_out
for v in 0 1; do
  BDFB_SPLIT_JAC_TPC=$v timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_jactpc$v.json 2> gpurun_out/bench_c4_jactpc$v.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_c4_jactpc$v.json').read().splitlines()[-1]);print('jac_tpc $v', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
done
BDFB_SPLIT_JAC_TPC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "flame_parity and split" 2>&1 | tail -1
