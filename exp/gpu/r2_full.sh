#!/bin/bash
# round 2: the full GPU suite, smoke(), and the bench under torchrun (1 rank: the NCCL plumbing path)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1
tail -4 gpurun_out/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
echo "torchrun rc=$?"; tail -c 300 gpurun_out/bench_torchrun1.json
