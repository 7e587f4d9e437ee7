# debug: CVDiag SPLIT vs oracle per-cell statistics on a small H2 flame field
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2405_01713_b200 as P
from synth import flame_field
from oracle import oracle as O
ls = sys.argv[1] if len(sys.argv) > 1 else "diag"
y0, rho, F, prog = flame_field("h2_lidryer", 16, dt=1e-6)
N = 512
y0, rho, F = y0[:, :N].copy(), rho[:N].copy(), F[:, :N].copy()
b = P.Batch(N, 10, 1e-6, 1e-10); b.set_model("h2"); b.set_linear_solver(ls)
cs = b.attach_cell_stats()
y = torch.tensor(y0, device="cuda"); b.integrate(0.0, 1e-6, y, f_ext=torch.tensor(F, device="cuda"), aux=torch.tensor(rho, device="cuda"))
st = b.stats(); sg = {k: v.cpu().numpy() for k, v in cs.items()}
yo, so = O.integrate_batch(O.Model.mechanism("h2_lidryer"), y0, 0, 1e-6, 1e-6, 1e-10, rho=rho, fext_yc=F, group=1, threads=8,
                           ls=O.LS_DIAG if ls == "diag" else O.LS_GMRES)
keys = ("nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn")
diff = [c for c in range(N) if any(sg[k][c] != so[k][c] for k in keys)]
print(ls, "cells with different stats", len(diff), "of", N, st)
for c in diff[:8]:
    print(c, "gpu", [int(sg[k][c]) for k in keys], "orc", [int(so[k][c]) for k in keys], "prog", prog[c])
err = np.abs(y.cpu().numpy() - yo) / (1e-6 * np.abs(yo) + 1e-10)
print("max err/tol", err.max())
