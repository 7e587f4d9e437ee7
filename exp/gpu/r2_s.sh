#!/bin/bash
# round 2 (session 3), final library (ATTEMPT unroll 1, chunks of 1 element): suite, smoke, default bench, reference arm, C5P, C4 dt 1e-7
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d.get("ms_per_step"), {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2s.log 2>&1
tail -3 gpurun_out/gpu_tests_r2s.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2s.log 2>&1; tail -1 gpurun_out/smoke_r2s.log | cut -c1-120
timeout 1200 python bench.py > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err
summ gpurun_out/bench_r2s.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r2s_reference.json 2> gpurun_out/bench_r2s_reference.err
tail -c 400 gpurun_out/bench_r2s_reference.json
timeout 900 python bench.py --config C5P --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2s_c5p.json 2> gpurun_out/bench_r2s_c5p.err
summ gpurun_out/bench_r2s_c5p.json
timeout 900 python bench.py --dt 1e-7 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r2s_dt1e-7.json 2> gpurun_out/bench_r2s_dt7.err
summ gpurun_out/bench_r2s_dt1e-7.json
