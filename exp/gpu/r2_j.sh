#!/bin/bash
# round 2 (session 3): the Jacobian diagnostic runs the two-pass K_jac code; suite; C4 launch list (2.1M-cell
# slab of the C4 field, every launch of one integrate); ncu --set full of one mid-run K_ctl and K_rhs (1M cells)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2j.log 2>&1
tail -3 gpurun_out/gpu_tests_r2j.log
grep -h "worst row-scaled" gpurun_out/gpu_tests_r2j.log | head; 
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -s -k "jacobian_parity" 2>&1 | grep -E "worst|passed|failed" | head -12
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_2M.csv \
  python exp/run_one.py drm19 128 split > gpurun_out/launches_c4_2M.log 2>&1
tail -2 gpurun_out/launches_c4_2M.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_ctl_kernel|split_rhs_kernel" \
  --launch-skip 200 --launch-count 2 -o gpurun_out/ncu_ctl_rhs_1M -f python exp/run_one.py drm19 100 split \
  > gpurun_out/ncu_ctl_rhs_1M.log 2>&1
tail -2 gpurun_out/ncu_ctl_rhs_1M.log
