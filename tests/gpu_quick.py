"""Quick GPU bring-up script (not a test module): runs each model small and compares with the oracle."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_01713_b200 as P
from oracle import oracle as O
from synth import flame_field, robertson_field, nyx_field
dev = torch.device("cuda", 0)

def report(name, yg, yo, rtol, atol, sg=None, so=None):
    tol = 10 * (rtol * np.abs(yo) + atol)
    err = np.abs(yg - yo) / tol
    bad = (err > 1).any(axis=0)
    msg = f"{name}: max err/tol10 {err.max():.3g} bad cells {bad.sum()}/{yg.shape[1]}"
    if sg is not None:
        same = np.mean([np.all([sg[k][c] == so[k][c] for k in ('nst','nfe','nje','nsetups','nni','netf','ncfn')]) for c in range(yg.shape[1])])
        msg += f" identical-stats frac {same:.3f} nst gpu/orc {sg['nst'].sum()}/{so['nst'].sum()}"
    print(msg, flush=True)

def run(model, mname, n, y0, t1, rtol, atol, rho=None, F=None, kernel="thread"):
    N = y0.shape[1]
    b = P.Batch(N, n, rtol, atol)
    b.set_kernel(kernel)
    b.set_model(model)
    group = b.wrms_group
    cs = b.attach_cell_stats()
    y = torch.tensor(y0, device=dev)
    b.integrate(0.0, t1, y, f_ext=None if F is None else torch.tensor(F, device=dev),
                aux=None if rho is None else torch.tensor(rho, device=dev))
    st = b.stats()
    print(model, kernel, "G", group, st, "kernel ms", b.last_kernel_ms(), flush=True)
    sg = {k: v.cpu().numpy() for k, v in cs.items()}
    m = O.Model.mechanism(mname) if mname not in ("robertson", "kwh", "linear") else (
        O.Model.robertson() if mname == "robertson" else (O.Model.nyx_kwh() if mname == "kwh" else O.Model.linear([-1.0])))
    t = time.time()
    yo, so = O.integrate_batch(m, y0, 0.0, t1, rtol, atol, rho=rho, fext_yc=F, group=group, threads=8)
    print(" oracle s", time.time() - t)
    report(model, y.cpu().numpy(), yo, rtol, atol, sg, so)
    return sg, so

steps = sys.argv[1:] or ["lu", "linear", "rob", "nyx", "h2", "drm"]
for s in steps:
    try:
        if s == "lu":
            for n in (1, 2, 3, 4, 5, 8, 10, 16, 22, 32):
                N = 1000
                rng = np.random.default_rng(n)
                M = rng.standard_normal((n, n, N)); bb = rng.standard_normal((n, N))
                LU, piv, x, info = P.lu_factor_solve(torch.tensor(M, device=dev), torch.tensor(bb, device=dev))
                LU, piv, x, info = LU.cpu().numpy(), piv.cpu().numpy(), x.cpu().numpy(), info.cpu().numpy()
                ok = 0
                for c in range(N):
                    LUo, pivo, io = O.lu_factor(M[:, :, c])
                    xo = O.lu_solve(LUo, pivo, bb[:, c])
                    ok += np.array_equal(pivo, piv[:, c]) and np.array_equal(LUo, LU[:, :, c]) and np.array_equal(xo, x[:, c])
                print("LU n", n, "bitwise identical", ok, "/", N, flush=True)
        if s == "linear":
            run("linear", "linear", 1, np.ones((1, 64)), 1.0, 1e-6, 1e-12)
        if s == "rob":
            run("robertson", "robertson", 3, robertson_field(1024), 40.0, 1e-4, 1e-8)
            run("robertson", "robertson", 3, robertson_field(1024), 40.0, 1e-6, 1e-10)
        if s == "nyx":
            e, rho, fe = nyx_field(16)
            run("nyx_kwh", "kwh", 1, e, 3e15, 1e-6, 1e-10, rho=rho, F=fe)
        if s == "h2":
            y, rho, F, prog = flame_field("h2_lidryer", 16)
            for k in ("thread", "group", "split"):
                run("h2", "h2_lidryer", 10, y, 1e-5, 1e-6, 1e-10, rho=rho, F=F, kernel=k)
        if s == "drm":
            y, rho, F, prog = flame_field("drm19_class", 16)
            for k in ("thread", "group", "split"):
                run("drm19", "drm19_class", 22, y, 1e-5, 1e-6, 1e-10, rho=rho, F=F, kernel=k)
        if s == "time":
            L = int(os.environ.get("L", "64"))
            y, rho, F, prog = flame_field("drm19_class", L)
            for k in os.environ.get("KS", "thread,split").split(","):
                b = P.Batch(y.shape[1], 22, 1e-6, 1e-10)
                b.set_kernel(k)
                b.set_model("drm19")
                yy = torch.tensor(y, device=dev)
                b.integrate(0.0, 1e-5, yy, f_ext=torch.tensor(F, device=dev), aux=torch.tensor(rho, device=dev))
                st = b.stats()
                ms = b.last_kernel_ms()
                print(f"time drm19 {k} L={L}: {ms:.1f} ms  {y.shape[1] / ms * 1e3:.3e} cells/s  {st}", flush=True)
    except Exception:
        traceback.print_exc()
