#!/bin/bash
# round 2: K_ctl without block barriers (warp-private shared state)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solvers.py -q -p no:cacheprovider -x -k "split or flame or gmres or cvdiag or gri53 or edge or c4" > gpurun_out/gpu_nobar.log 2>&1; tail -1 gpurun_out/gpu_nobar.log
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4_nobar.json 2> gpurun_out/bench_c4_nobar.err
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_nobar.json').read().splitlines()[-1]);print('C4', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
