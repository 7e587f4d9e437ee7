#!/bin/bash
# round 2 (session 3): ATTEMPT chunk of 1 element (exp/lib_ch1.so) and error-test norm unroll 2 (exp/lib_err2.so)
# vs the main library, same box, two runs each
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
for v in ch1 err2; do
  [ -f exp/lib_$v.so ] && BDFB_LIB=exp/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
    -k "(flame_parity and split) or slot_reuse" > gpurun_out/gpu_tests_$v.log 2>&1 && tail -1 gpurun_out/gpu_tests_$v.log
done
for r in 1 2; do
  timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r_main$r.json 2> /dev/null
  summ gpurun_out/bench_r_main$r.json
  for v in ch1 err2; do
    [ -f exp/lib_$v.so ] || continue
    BDFB_LIB=exp/lib_$v.so timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r_${v}_$r.json 2> /dev/null
    summ gpurun_out/bench_r_${v}_$r.json
  done
done
