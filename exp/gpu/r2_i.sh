#!/bin/bash
# round 2 (session 3): jac_sum takes the per-species thermo (balanced parts); the two-pass generated Jacobian for
# the 53-species mechanism too (C5P); suite, C4 bench, C5P bench with A/B vs the lanes Jacobian
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2i.log 2>&1
tail -3 gpurun_out/gpu_tests_r2i.log
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in d.get("phases", {}).items()})
PYEOF
}
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err
summ gpurun_out/bench_r2i.json
timeout 900 python bench.py --config C5P --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2i_c5p.json 2> gpurun_out/bench_r2i_c5p.err
summ gpurun_out/bench_r2i_c5p.json
BDFB_SPLIT_JAC2=0 timeout 900 python bench.py --config C5P --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2i_c5p_lanes.json 2> gpurun_out/bench_r2i_c5p_lanes.err
summ gpurun_out/bench_r2i_c5p_lanes.json
