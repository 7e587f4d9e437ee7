"""Small invocations of every kernel family through the C ABI, for compute-sanitizer (memcheck / racecheck /
synccheck) runs on the B200 box: SPLIT dense / CVDiag / GMRES (H2, DRM19, n = 54), ERK, THREAD, GROUP, the
persistent small-model kernels, the global-norm mode (DRM19, n = 54), typical-value reductions, diagnostics."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_01713_b200 as P  # noqa: E402
from synth import flame_field, robertson_field, nyx_field  # noqa: E402

dev = torch.device("cuda", 0)


def cu(a):
    return None if a is None else torch.tensor(np.ascontiguousarray(a), device=dev)


def run(name, n, mech, L, dt, kernel="auto", ls=None, method=None, mode=P.MODE_PER_CELL):
    y0, rho, F, _ = flame_field(mech, L, dt=dt)
    b = P.Batch(y0.shape[1], n, 1e-6, 1e-10, mode=mode, mxstep=200000)
    b.set_kernel(kernel)
    b.set_model(name)
    if ls:
        b.set_linear_solver(ls)
    if method:
        b.set_method(method)
    y = cu(y0)
    b.integrate(0.0, dt, y, f_ext=cu(F), aux=cu(rho))
    st = b.stats()
    print(name, kernel, ls, method, mode, st["n_failed"], st["nst"], flush=True)


run("h2", 10, "h2_lidryer", 4, 1e-6)
run("drm19", 22, "drm19_class", 4, 1e-6)
run("drm19", 22, "drm19_class", 4, 1e-6, ls="diag")
run("drm19", 22, "drm19_class", 4, 1e-6, ls="gmres")
run("drm19", 22, "drm19_class", 4, 1e-7, method="erk4")
run("h2", 10, "h2_lidryer", 4, 1e-6, kernel="thread")
run("h2", 10, "h2_lidryer", 4, 1e-6, kernel="group")
run("gri53", 54, "gri53_class", 3, 1e-7)
run("gri53", 54, "gri53_class", 3, 1e-7, ls="gmres")
run("drm19", 22, "drm19_class", 4, 1e-6, mode=P.MODE_GLOBAL_NORM)
run("gri53", 54, "gri53_class", 3, 1e-7, mode=P.MODE_GLOBAL_NORM)
yr = robertson_field(64)
b = P.Batch(64, 3, 1e-6, 1e-10)
b.set_model("robertson")
y = cu(yr)
b.integrate(0.0, 1.0, y)
e, rho, fe = nyx_field(8, dt=3e15)
b = P.Batch(e.shape[1], 1, 1e-6, 1e-10)
b.set_model("nyx_kwh")
y = cu(e)
b.integrate(0.0, 3e15, y, f_ext=cu(fe), aux=cu(rho))
yf, rho, F, _ = flame_field("drm19_class", 4)
b = P.Batch(yf.shape[1], 22, 1e-6, 1e-10)
b.set_model("drm19")
lo, hi = b.minmax(cu(yf))
f, st = P.eval_rhs(b, cu(yf), f_ext=cu(F), aux=cu(rho))
torch.cuda.synchronize()
print("sanitize run done", flush=True)
