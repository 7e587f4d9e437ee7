#!/bin/bash
./exp/tpc/tpc_bench
python - <<'PY'
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2405_01713_b200 as P
N = 1 << 20
y = torch.full((22, N), 1.0 / 21, dtype=torch.float64, device='cuda'); y[21] = 1200 + torch.arange(N, device='cuda') % 1000
rho = torch.full((N,), 2.4e-4, dtype=torch.float64, device='cuda')
b = P.Batch(N, 22, 1e-6, 1e-10); b.set_model('drm19')
P.eval_rhs(b, y, aux=rho); torch.cuda.synchronize()
t = time.time(); reps = 20
for _ in range(reps): P.eval_rhs(b, y, aux=rho)
torch.cuda.synchronize(); dt = time.time() - t
print(f"warp-cooperative RHS: {N*reps/dt:.3e} RHS/s")
PY
