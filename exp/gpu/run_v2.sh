#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v2_pytest.log 2>&1
echo "rc $?" >> gpurun_out/v2_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2_smoke.log 2>&1
echo "smoke rc $?" >> gpurun_out/v2_smoke.log
timeout 900 python bench.py > gpurun_out/v2_C4.json 2> gpurun_out/v2_C4.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v2_ref.json 2> gpurun_out/v2_ref.err
