#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py -q -p no:cacheprovider -k gri53 2>&1 | tail -1
timeout 900 python bench.py --config C5P --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c5p_jac.json 2> gpurun_out/bench_c5p_jac.err
python -c "import json;d=json.loads(open('gpurun_out/bench_c5p_jac.json').read().splitlines()[-1]);print('C5P', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
