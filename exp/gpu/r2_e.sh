#!/bin/bash
# round 2 (session 3): K_rhs runs the Newton residual + LU solve (RV_SOLVED), warp-uniform full-mask K_lu;
# full GPU suite, default bench; then the slot-major VEC variant (exp/lib_vecaos.so): parity subset + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2e.log 2>&1
tail -3 gpurun_out/gpu_tests_r2e.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err
tail -c 300 gpurun_out/bench_r2e.json
python - <<'EOF'
import json
d = json.loads(open("gpurun_out/bench_r2e.json").read().strip().splitlines()[-1])
print("C4", d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in d["phases"].items()})
EOF
if [ -f exp/lib_vecaos.so ]; then
  BDFB_LIB=exp/lib_vecaos.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
    -k "split_lu or (flame_parity and split) or slot_reuse or full_size_c4" > gpurun_out/gpu_tests_vecaos.log 2>&1
  tail -2 gpurun_out/gpu_tests_vecaos.log
  BDFB_LIB=exp/lib_vecaos.so timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_vecaos.json 2> gpurun_out/bench_vecaos.err
  python - <<'EOF'
import json
d = json.loads(open("gpurun_out/bench_vecaos.json").read().strip().splitlines()[-1])
print("C4 vecaos", d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in d["phases"].items()})
EOF
fi
