#!/bin/bash
# round 2 (session 3), final state: suite, smoke, default bench with the CPU baseline, C5P A/B for the n = 54 LU
# block size (exp/lib_glu192.so: two 192-thread blocks per SM), ncu --set full of one mid-run K_ctl (CSV on the box)
mkdir -p gpurun_out
summ() {
python - "$1" <<'PYEOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], {k: round(v["ms"], 1) for k, v in (d.get("phases") or {}).items()})
PYEOF
}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2m.log 2>&1
tail -3 gpurun_out/gpu_tests_r2m.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2m.log 2>&1; tail -1 gpurun_out/smoke_r2m.log | cut -c1-200
timeout 1200 python bench.py > gpurun_out/bench_r2m.json 2> gpurun_out/bench_r2m.err
summ gpurun_out/bench_r2m.json
timeout 900 python bench.py --config C5P --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2m_c5p.json 2> gpurun_out/bench_r2m_c5p.err
summ gpurun_out/bench_r2m_c5p.json
if [ -f exp/lib_glu192.so ]; then
  BDFB_LIB=exp/lib_glu192.so timeout 900 python bench.py --config C5P --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_r2m_c5p_glu192.json 2> gpurun_out/bench_r2m_c5p_glu192.err
  summ gpurun_out/bench_r2m_c5p_glu192.json
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_ctl_kernel" \
  --launch-skip 100 --launch-count 1 -o /tmp/ncu_ctl_1M -f python exp/run_one.py drm19 100 split \
  > gpurun_out/ncu_ctl_1M_m.log 2>&1
ncu -i /tmp/ncu_ctl_1M.ncu-rep --page raw --csv > gpurun_out/ncu_ctl_1M_m_raw.csv 2>&1
ncu -i /tmp/ncu_ctl_1M.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_ctl_1M_m_source.csv 2>&1
python exp/ncu_lines.py gpurun_out/ncu_ctl_1M_m_source.csv 45 > gpurun_out/ncu_ctl_1M_m_by_line.txt 2>&1
gzip -f gpurun_out/ncu_ctl_1M_m_source.csv
head -12 gpurun_out/ncu_ctl_1M_m_by_line.txt | cut -c1-160
