#!/bin/bash
# round 2: the 53-species mechanism per cell (SPLIT n = 54, GMRES, ERK): parity + a C5P bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solvers.py -q -s -p no:cacheprovider -k gri53 > gpurun_out/gpu_gri_pc.log 2>&1
grep -E "identical|passed|failed|Error" gpurun_out/gpu_gri_pc.log | head -20
timeout 1500 python bench.py --config C5P --steps 3 --warmup 3 > gpurun_out/bench_c5p.json 2> gpurun_out/bench_c5p.err
tail -3 gpurun_out/bench_c5p.err
python -c "import json;d=json.loads(open('gpurun_out/bench_c5p.json').read().splitlines()[-1]);print('C5P', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['whole_step']['frac'], {k:round(x['ms']) for k,x in d['phases'].items()})"
