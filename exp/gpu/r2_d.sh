#!/bin/bash
# round 2 (session 3): full GPU suite on the restored tree, default bench line, ncu --set full of one mid-run
# launch each of K_lu and K_jac (1M-cell C4 field, SPLIT)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2d.log 2>&1
tail -3 gpurun_out/gpu_tests_r2d.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err
tail -c 600 gpurun_out/bench_r2d.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_lu_kernel|split_jac_kernel" \
  --launch-skip 200 --launch-count 2 -o gpurun_out/ncu_setup_1M -f python exp/run_one.py drm19 100 split \
  > gpurun_out/ncu_setup_1M.log 2>&1
tail -3 gpurun_out/ncu_setup_1M.log
