"""Profiling helper: one integrate of a flame field (mech, L, kernel) -- for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_01713_b200 as P
from synth import flame_field
mech = sys.argv[1] if len(sys.argv) > 1 else "drm19"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 48
kernel = sys.argv[3] if len(sys.argv) > 3 else "thread"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
name, n = {"drm19": ("drm19_class", 22), "h2": ("h2_lidryer", 10)}[mech]
y, rho, F, prog = flame_field(name, L)
dev = torch.device("cuda", 0)
b = P.Batch(y.shape[1], n, 1e-6, 1e-10)
b.set_kernel(kernel)
b.set_model(mech)
for r in range(reps):
    yy = torch.tensor(y, device=dev)
    b.integrate(0.0, 1e-5, yy, f_ext=torch.tensor(F, device=dev), aux=torch.tensor(rho, device=dev))
    st = b.stats()
    print(mech, kernel, L, b.last_kernel_ms(), "ms", st, flush=True)
