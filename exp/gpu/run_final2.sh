#!/bin/bash
# final round-1 verification: GPU tests, smoke, default bench line, reference arm, and the ncu launch list of the
# bench workload at full size (C4, 256^3; --steps 1 --warmup 0 --no-cpu to bound the ncu time)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/z2_pytest.log 2>&1
echo "rc $?" >> gpurun_out/z2_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z2_smoke.log 2>&1
echo "smoke rc $?" >> gpurun_out/z2_smoke.log
timeout 900 python bench.py > gpurun_out/z2_C4.json 2> gpurun_out/z2_C4.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z2_launches_full.csv \
    python bench.py --no-cpu --steps 1 --warmup 0 > gpurun_out/z2_l.log 2>&1
