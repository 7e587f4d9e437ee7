#!/bin/bash
# round 2 (session 3): K_ctl resident blocks capped at 2 per SM (8 warps, same binary, BDFB_SPLIT_CTL_SMEM=80000:
# more L1 per warp) vs 3 (12 warps)
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
for r in 1 2; do
  timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_u_main$r.json 2> /dev/null
  summ gpurun_out/bench_u_main$r.json
  BDFB_SPLIT_CTL_SMEM=80000 timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_u_2blk_$r.json 2> /dev/null
  summ gpurun_out/bench_u_2blk_$r.json
done
