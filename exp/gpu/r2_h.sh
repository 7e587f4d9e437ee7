#!/bin/bash
# round 2 (session 3): K_lu pivot-row picks with R-1 selects; K_jac pass 1 parted (4 warp-uniform parts + jac_sum);
# two-pass K_jac with a warp-blocked SoA scratch; suite, bench, A/B vs the group Jacobian, ncu of K_lu + K_jac passes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2h.log 2>&1
tail -3 gpurun_out/gpu_tests_r2h.log
summ() {
python - "$1" <<'EOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in d["phases"].items()})
EOF
}
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r2h.json 2> gpurun_out/bench_r2h.err
summ gpurun_out/bench_r2h.json
BDFB_SPLIT_JAC2=0 timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2h_jaclanes.json 2> gpurun_out/bench_r2h_jaclanes.err
summ gpurun_out/bench_r2h_jaclanes.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_lu_kernel|split_jac_" \
  --launch-skip 400 --launch-count 4 -o gpurun_out/ncu_setup4_1M -f python exp/run_one.py drm19 100 split \
  > gpurun_out/ncu_setup4_1M.log 2>&1
tail -2 gpurun_out/ncu_setup4_1M.log
