#!/bin/bash
mkdir -p gpurun_out
for cfg in C5P C4; do
BDFB_LIB=exp/lib_minb2.so timeout 900 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_minb2_$cfg.json 2> gpurun_out/bench_minb2_$cfg.err
python -c "import json;d=json.loads(open('gpurun_out/bench_minb2_$cfg.json').read().splitlines()[-1]);print('minb2 $cfg', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
done
