#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/last_pytest.log 2>&1
echo "rc $?" >> gpurun_out/last_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1
echo "smoke rc $?" >> gpurun_out/last_smoke.log
timeout 900 python bench.py > gpurun_out/last_C4.json 2> gpurun_out/last_C4.err
