# debug: CVDiag SPLIT vs oracle, step by step via mxstep = k (TOO_MUCH_WORK returns the k-step state)
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2405_01713_b200 as P
from synth import flame_field
from oracle import oracle as O
y0, rho, F, prog = flame_field("h2_lidryer", 16, dt=1e-6)
cells = [3, 4]
y0, rho, F = np.ascontiguousarray(y0[:, cells]), rho[cells].copy(), np.ascontiguousarray(F[:, cells])
N = len(cells)
keys = ("nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn")
for k in range(1, 40):
    b = P.Batch(N, 10, 1e-6, 1e-10, mxstep=k); b.set_model("h2"); b.set_linear_solver("diag")
    cs = b.attach_cell_stats()
    y = torch.tensor(y0, device="cuda"); b.integrate(0.0, 1e-6, y, f_ext=torch.tensor(F, device="cuda"), aux=torch.tensor(rho, device="cuda"))
    sg = {kk: v.cpu().numpy() for kk, v in cs.items()}
    yo, so = O.integrate_batch(O.Model.mechanism("h2_lidryer"), y0, 0, 1e-6, 1e-6, 1e-10, rho=rho, fext_yc=F, group=1,
                               ls=O.LS_DIAG, mxstep=k)
    yg = y.cpu().numpy()
    for c in range(N):
        d = [int(sg[kk][c]) for kk in keys], [int(so[kk][c]) for kk in keys]
        same = d[0] == d[1] and np.array_equal(yg[:, c], yo[:, c])
        if not same:
            print("k", k, "cell", cells[c], "gpu", d[0], "orc", d[1], "h", sg["h_last"][c], so["h_last"][c],
                  "t", sg["t_reached"][c], so["t_reached"][c], "maxrel", np.max(np.abs(yg[:, c] - yo[:, c]) / (np.abs(yo[:, c]) + 1e-30)))
