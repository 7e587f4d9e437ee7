#!/bin/bash
# round 2 (session 3): ATTEMPT-pass chunks in flight 2 (default) vs 4 (exp/lib_unroll4.so), same box
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
BDFB_LIB=exp/lib_unroll4.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
  -k "(flame_parity and split) or slot_reuse or full_size_c4" > gpurun_out/gpu_tests_unroll4.log 2>&1
tail -1 gpurun_out/gpu_tests_unroll4.log
for r in 1 2; do
  timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_o_main$r.json 2> /dev/null
  summ gpurun_out/bench_o_main$r.json
  BDFB_LIB=exp/lib_unroll4.so timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_o_unroll4_$r.json 2> /dev/null
  summ gpurun_out/bench_o_unroll4_$r.json
done
