#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py -q -p no:cacheprovider -k "gmres" 2>&1 | tail -1
timeout 1200 python bench.py --config C4 --ls gmres --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_gmres2.json 2> gpurun_out/bench_c4_gmres2.err
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_gmres2.json').read().splitlines()[-1]);print('gmres', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
