#!/bin/bash
# round 2 (session 3): compute-sanitizer memcheck + racecheck over every kernel family with the final build (new
# K_lu, two-pass K_jac, n = 54 K_lu shape, global-norm generated J); ATTEMPT unroll 1 vs 2 (exp/lib_unroll1.so)
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python exp/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run done" gpurun_out/sanitize_$tool.log | tail -3
done
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
if [ -f exp/lib_unroll1.so ]; then
  for r in 1 2; do
    timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_p_main$r.json 2> /dev/null
    summ gpurun_out/bench_p_main$r.json
    BDFB_LIB=exp/lib_unroll1.so timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_p_unroll1_$r.json 2> /dev/null
    summ gpurun_out/bench_p_unroll1_$r.json
  done
fi
