#!/bin/bash
# round 2 (session 3): cell load/store and the cvHin preamble issue their loads before their stores; the
# global-norm n = 54 J from the generated two-pass Jacobian; suite, C4, C5 (A/B BDFB_GLOBAL_JAC2=0), K_ctl by line
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2l.log 2>&1
tail -3 gpurun_out/gpu_tests_r2l.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r2l.json 2> gpurun_out/bench_r2l.err
summ gpurun_out/bench_r2l.json
timeout 1200 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2l_c5.json 2> gpurun_out/bench_r2l_c5.err
summ gpurun_out/bench_r2l_c5.json
BDFB_GLOBAL_JAC2=0 timeout 1200 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2l_c5_lanes.json 2> gpurun_out/bench_r2l_c5_lanes.err
summ gpurun_out/bench_r2l_c5_lanes.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_ctl_kernel" \
  --launch-skip 100 --launch-count 1 -o /tmp/ncu_ctl_1M -f python exp/run_one.py drm19 100 split \
  > gpurun_out/ncu_ctl_1M_l.log 2>&1
ncu -i /tmp/ncu_ctl_1M.ncu-rep --page raw --csv > gpurun_out/ncu_ctl_1M_l_raw.csv 2>&1
ncu -i /tmp/ncu_ctl_1M.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_ctl_1M_l_source.csv 2>&1
python exp/ncu_lines.py gpurun_out/ncu_ctl_1M_l_source.csv 45 > gpurun_out/ncu_ctl_1M_l_by_line.txt 2>&1
gzip -f gpurun_out/ncu_ctl_1M_l_source.csv
head -25 gpurun_out/ncu_ctl_1M_l_by_line.txt | cut -c1-160
