"""Diagnostic: end-state agreement of the Eq. 7 typical-atol integration (GPU SPLIT vs oracle) for several eta."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_01713_b200 as P
from oracle import oracle as O
from synth import flame_field
dev = torch.device("cuda", 0)
for mech, name, n in (("h2_lidryer", "h2", 10), ("drm19_class", "drm19", 22)):
    y0, rho, F, prog = flame_field(mech, 16, dt=1e-5)
    for eta in (1e-10, 1e-8, 1e-6):
        b = P.Batch(y0.shape[1], n, 1e-6, 1e-10)
        b.set_model(name)
        cs = b.attach_cell_stats()
        yd = torch.tensor(y0, device=dev)
        b.set_typical_atol(yd, eta=eta)
        b.integrate(0.0, 1e-5, yd, f_ext=torch.tensor(F, device=dev), aux=torch.tensor(rho, device=dev))
        atol = O.atol_from_typical(O.typical_values(y0), eta, 1e-30)
        yo, so = O.integrate_batch(O.Model.mechanism(mech), y0, 0.0, 1e-5, 1e-6, atol, rho=rho, fext_yc=F,
                                   group=b.wrms_group, threads=8)
        yg = yd.cpu().numpy()
        r = np.abs(yg - yo) / (10 * (1e-6 * np.abs(yo) + atol[:, None]))
        same = np.mean([all(cs[k].cpu().numpy()[c] == so[k][c] for k in ("nst", "nfe", "nsetups", "netf")) for c in range(y0.shape[1])])
        print(name, eta, "max ratio", r.max(), "bad cells", (r > 1).any(axis=0).sum(), "of", y0.shape[1], "same stats", same, flush=True)
