#!/bin/bash
# round 2: ERK in the SPLIT organisation (K_erk + K_rhs) vs the persistent kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py -q -s -p no:cacheprovider -k erk > gpurun_out/gpu_erksplit.log 2>&1; grep -E "identical|passed|failed" gpurun_out/gpu_erksplit.log | tail -8
timeout 900 python bench.py --config C4 --method erk4 --dt 1e-7 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_erk_split.json 2> gpurun_out/bench_erk_split.err
tail -2 gpurun_out/bench_erk_split.err
python -c "import json;d=json.loads(open('gpurun_out/bench_erk_split.json').read().splitlines()[-1]);print('erk split', d['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['whole_step']['frac'], {k:round(x['ms']) for k,x in d['phases'].items()})"
