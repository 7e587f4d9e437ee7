#!/bin/bash
# round 2 (session 3): n = 54 K_lu two 192-thread blocks per SM by default; K_lu shared-memory pivot-row
# publication A/B (exp/lib_lusmem.so); suite, C5P, default bench (CPU baseline 120K cells)
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2n.log 2>&1
tail -3 gpurun_out/gpu_tests_r2n.log
timeout 900 python bench.py --config C5P --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2n_c5p.json 2> gpurun_out/bench_r2n_c5p.err
summ gpurun_out/bench_r2n_c5p.json
if [ -f exp/lib_lusmem.so ]; then
  BDFB_LIB=exp/lib_lusmem.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
    -k "split_lu or (flame_parity and split) or slot_reuse" > gpurun_out/gpu_tests_lusmem.log 2>&1
  tail -1 gpurun_out/gpu_tests_lusmem.log
  BDFB_LIB=exp/lib_lusmem.so timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_lusmem.json 2> gpurun_out/bench_lusmem.err
  summ gpurun_out/bench_lusmem.json
fi
timeout 1200 python bench.py > gpurun_out/bench_r2n.json 2> gpurun_out/bench_r2n.err
summ gpurun_out/bench_r2n.json
python -c "import json; d=json.loads(open('gpurun_out/bench_r2n.json').read().strip().splitlines()[-1]); print(d['cpu_baseline']['value'], d['cpu_baseline']['passes_s'], d['e2e']['value'], d['clocks'])"
