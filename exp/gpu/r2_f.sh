#!/bin/bash
# round 2 (session 3): two-pass generated K_jac (split_jac_p1/p2), full-mask K_lu, fused K_rhs solve off;
# full GPU suite, default bench, group-Jacobian A/B, ncu --set full of K_lu and the two K_jac passes (1M cells)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2f.log 2>&1
tail -3 gpurun_out/gpu_tests_r2f.log
summ() {
python - "$1" <<'EOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in d["phases"].items()})
EOF
}
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err
summ gpurun_out/bench_r2f.json
BDFB_SPLIT_JAC2=0 timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2f_jaclanes.json 2> gpurun_out/bench_r2f_jaclanes.err
summ gpurun_out/bench_r2f_jaclanes.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_lu_kernel|split_jac_p" \
  --launch-skip 300 --launch-count 3 -o gpurun_out/ncu_setup2_1M -f python exp/run_one.py drm19 100 split \
  > gpurun_out/ncu_setup2_1M.log 2>&1
tail -2 gpurun_out/ncu_setup2_1M.log
