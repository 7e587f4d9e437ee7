#!/bin/bash
# round 2 (session 3): set_bdf / prepare_next inlined in K_ctl (exp/lib_hotinl.so) A/B; C4 at dt 1e-7 (BDF);
# C4 launch list (2.1M-cell slab, every launch of one integrate) summarised on the box; ncu --set full of one
# mid-run K_ctl and K_rhs (1M cells) exported to CSV on the box (the .ncu-rep with source exceeds the 64 MiB cap)
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in d.get("phases", {}).items()})
PYEOF
}
BDFB_LIB=exp/lib_hotinl.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
  -k "(flame_parity and split) or slot_reuse" > gpurun_out/gpu_tests_hotinl.log 2>&1
tail -1 gpurun_out/gpu_tests_hotinl.log
BDFB_LIB=exp/lib_hotinl.so timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_hotinl.json 2> gpurun_out/bench_hotinl.err
summ gpurun_out/bench_hotinl.json
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2k.json 2> gpurun_out/bench_r2k.err
summ gpurun_out/bench_r2k.json
timeout 900 python bench.py --dt 1e-7 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4_bdf_dt1e-7_r2k.json 2> gpurun_out/bench_dt7.err
summ gpurun_out/bench_c4_bdf_dt1e-7_r2k.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_2M.csv \
  python exp/run_one.py drm19 128 split > gpurun_out/launches_c4_2M.log 2>&1
python exp/launch_summary.py gpurun_out/launches_c4_2M.csv > gpurun_out/launches_c4_2M_summary.txt 2>&1
head -30 gpurun_out/launches_c4_2M_summary.txt
gzip -f gpurun_out/launches_c4_2M.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_ctl_kernel|split_rhs_kernel" \
  --launch-skip 200 --launch-count 2 -o /tmp/ncu_ctl_rhs_1M -f python exp/run_one.py drm19 100 split \
  > gpurun_out/ncu_ctl_rhs_1M.log 2>&1
ncu -i /tmp/ncu_ctl_rhs_1M.ncu-rep --page raw --csv > gpurun_out/ncu_ctl_rhs_1M_raw.csv 2>&1
ncu -i /tmp/ncu_ctl_rhs_1M.ncu-rep --page source --csv --print-source cuda,sass -k regex:split_ctl_kernel \
  > gpurun_out/ncu_ctl_1M_source.csv 2>&1
python exp/ncu_lines.py gpurun_out/ncu_ctl_1M_source.csv 45 > gpurun_out/ncu_ctl_1M_by_line.txt 2>&1
gzip -f gpurun_out/ncu_ctl_1M_source.csv
ls -la gpurun_out | tail -12
