#!/bin/bash
# round 2: register-row LU for the n = 54 global-norm path (gl_lu): parity + C5 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "global_norm or gri53 or rhs_parity or lu" > gpurun_out/gpu_c5lu.log 2>&1; tail -2 gpurun_out/gpu_c5lu.log
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5_lu.json 2> gpurun_out/bench_c5_lu.err
python -c "import json;d=json.loads(open('gpurun_out/bench_c5_lu.json').read().splitlines()[-1]);print('C5', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['fp64']['whole_step']['frac'])"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches_lu.csv python bench.py --config C5 --cells 262144 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
python exp/launch_summary.py gpurun_out/c5_launches_lu.csv | head -8
