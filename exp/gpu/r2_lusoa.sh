#!/bin/bash
# round 2: warp-blocked SoA LU records (coalesced Newton-solve loads in K_ctl): parity + C4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "split_lu or flame_parity or lu_bit or full_size_c4" > gpu_lusoa.log 2>&1; tail -2 gpu_lusoa.log; cp gpu_lusoa.log gpurun_out/
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4_lusoa.json 2> gpurun_out/bench_c4_lusoa.err
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_lusoa.json').read().splitlines()[-1]);print('C4', d['value'], {k:round(x['ms']) for k,x in d['phases'].items()})"
