#!/bin/bash
# round 2 (session 3): K_ctl at 128 registers x 16 warps/SM (exp/lib_minb4.so, BDFB_SPLIT_CTL_MINB=4) vs 168 x 12
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
BDFB_LIB=exp/lib_minb4.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
  -k "(flame_parity and split) or slot_reuse or full_size_c4" > gpurun_out/gpu_tests_minb4.log 2>&1
tail -1 gpurun_out/gpu_tests_minb4.log
for r in 1 2; do
  timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_t_main$r.json 2> /dev/null
  summ gpurun_out/bench_t_main$r.json
  BDFB_LIB=exp/lib_minb4.so timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_t_minb4_$r.json 2> /dev/null
  summ gpurun_out/bench_t_minb4_$r.json
done
