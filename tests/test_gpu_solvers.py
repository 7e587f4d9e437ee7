"""GPU parity of the matrix-free linear solvers (CVDiag; inexact Newton-Krylov GMRES,
approaches 1A/1B, row f3) and of the explicit ERK (row f4): the CUDA path through the
C ABI vs the CPU oracle on identical seeded inputs.  Bar: end states |dy| <= 10 (rtol |y| + atol) per cell and
component (north_star), per-cell statuses equal, aggregate counters close."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2405_01713_b200 as P  # noqa: E402
from synth import flame_field  # noqa: E402

DEV = torch.device("cuda", 0)
STAT_KEYS = ("nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn")
MECH = {"h2": ("h2_lidryer", 10), "drm19": ("drm19_class", 22)}


def cu(a):
    return None if a is None else torch.tensor(np.ascontiguousarray(a), device=DEV)


def end_state_check(yg, yo, rtol, atol):
    tol = 10.0 * (rtol * np.abs(yo) + atol)
    err = np.abs(yg - yo)
    ok = err <= tol
    assert ok.all(), f"{(~ok.all(axis=0)).sum()} cells outside 10 tol; worst {np.max(err / tol):.3g}"


def envelope_check(yg, sg, oracle, model, y0, dt, rho, F, **kw):
    """Parity bar for configurations whose results are ill-conditioned with respect to rounding (CVDiag on
    coupled chemistry; GMRES with a small Krylov cap), reading R31: there the oracle itself,
    re-run with the listing's plain arithmetic (libm roots, true division: ulp-level changes), moves end
    states by up to ~10^3 x the 10 (rtol|y| + atol) band.  The CUDA path must then stay inside the oracle's
    own rounding envelope: equal statuses; a fraction of cells within the band no smaller than the oracle's
    (less 5 points); 99th percentile and maximum deviation at most 3x (+1 band) the oracle's."""
    ya, sa = oracle.integrate_batch(model, y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F, threads=16, **kw)
    yb, _ = oracle.integrate_batch(model, y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F, threads=16, plain=True,
                                   **kw)
    band = 10.0 * (1e-6 * np.abs(ya) + 1e-10)
    g = (np.abs(yg - ya) / band).max(axis=0)
    o = (np.abs(yb - ya) / band).max(axis=0)
    print(f"envelope: within band gpu {np.mean(g <= 1):.4f} oracle {np.mean(o <= 1):.4f}; q99 {np.quantile(g, 0.99):.3g}"
          f" vs {np.quantile(o, 0.99):.3g}; max {g.max():.3g} vs {o.max():.3g}")
    assert np.array_equal(sg["status"], sa["status"])
    assert np.mean(g <= 1) >= np.mean(o <= 1) - 0.05
    assert np.quantile(g, 0.99) <= 3 * np.quantile(o, 0.99) + 1
    assert g.max() <= 3 * o.max() + 1
    return sa


def run_ls(name, y0, dt, rho, F, ls, maxl=0, mxstep=10000):
    mech, n = MECH[name]
    b = P.Batch(y0.shape[1], n, 1e-6, 1e-10, mxstep=mxstep)
    b.set_model(name)
    b.set_linear_solver(ls, maxl)
    cs = b.attach_cell_stats()
    y = cu(y0)
    b.integrate(0.0, dt, y, f_ext=cu(F), aux=cu(rho))
    st = b.stats()
    return y.cpu().numpy(), {k: v.cpu().numpy() for k, v in cs.items()}, st, b.wrms_group


@pytest.mark.parametrize("name,dt", [("h2", 1e-6), ("h2", 1e-5), ("drm19", 1e-6), ("drm19", 1e-5)])
def test_gmres_parity(oracle, name, dt):
    """Inexact Newton-Krylov (maxl = 5): the strict north_star bar, 10 (rtol|y| + atol) on every cell."""
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 16, dt=dt)
    yg, sg, st, group = run_ls(name, y0, dt, rho, F, "gmres")
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F,
                                    group=group, threads=8, ls=oracle.LS_GMRES)
    assert st["n_failed"] == 0 and np.array_equal(sg["status"], so["status"])
    end_state_check(yg, yo, 1e-6, 1e-10)
    same = np.mean([all(sg[k][c] == so[k][c] for k in STAT_KEYS) for c in range(y0.shape[1])])
    print(f"{name} dt={dt} gmres: identical per-cell stats {same:.4f}; nli gpu {st['nli']} oracle {so['nli'].sum()}")
    assert same > 0.9
    assert st["nje"] == 0 and st["nsetups"] == 0
    assert abs(st["nli"] - so["nli"].sum()) <= 0.02 * so["nli"].sum()
    # the Newton-Krylov end states agree with the dense direct (2A) run to <= 100 rtol
    yd, _ = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho,
                                   fext_yc=F, group=group, threads=8)
    assert np.all(np.abs(yg - yd) <= 100 * (1e-6 * np.abs(yd) + 1e-10))


@pytest.mark.parametrize("name,dt", [("h2", 1e-6), ("h2", 1e-5), ("drm19", 1e-6), ("drm19", 1e-5)])
def test_cvdiag_parity(oracle, name, dt):
    """CVDiag on coupled chemistry: (a) the first steps, before rounding differences are amplified,
    agree with the oracle to 1e-9 relative with identical counters; (b) end states inside the oracle's own
    rounding envelope (envelope_check, reading R31)."""
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 16, dt=dt)
    m = oracle.Model.mechanism(mech)
    for k in (1, 2, 3):
        yg, sg, st, group = run_ls(name, y0, dt, rho, F, "diag", mxstep=k)
        yo, so = oracle.integrate_batch(m, y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F, group=group, threads=8,
                                        ls=oracle.LS_DIAG, mxstep=k)
        same = np.mean([all(sg[kk][c] == so[kk][c] for kk in STAT_KEYS) for c in range(y0.shape[1])])
        rel = np.abs(yg - yo) / (np.abs(yo) + 1e-10)
        print(f"{name} dt={dt} diag k={k}: identical stats {same:.4f}, max rel {rel.max():.3g}")
        assert same >= 0.99 and np.quantile(rel.max(axis=0), 0.99) <= 1e-9
    yg, sg, st, group = run_ls(name, y0, dt, rho, F, "diag")
    assert st["nje"] == st["nsetups"] and st["nli"] == 0
    envelope_check(yg, sg, oracle, m, y0, dt, rho, F, ls=oracle.LS_DIAG, group=group)


@pytest.mark.parametrize("ls", ["diag", "gmres"])
def test_matrix_free_slot_reuse(oracle, ls, monkeypatch):
    """64 slots for 4096 cells: records are reused many times (the GMRES basis, CVDiag's M^-1 and the nli
    counter of a previous cell must not leak): bit-identical to the one-cell-per-slot run."""
    monkeypatch.setenv("BDFB_SPLIT_SLOTS", "64")
    y0, rho, F, prog = flame_field("h2_lidryer", 16, dt=1e-5)
    yg, sg, st, group = run_ls("h2", y0, 1e-5, rho, F, ls)
    monkeypatch.delenv("BDFB_SPLIT_SLOTS")
    y2, s2, st2, _ = run_ls("h2", y0, 1e-5, rho, F, ls)
    assert np.array_equal(y2, yg) and st2 == st   # the pool size never changes a result
    if ls == "gmres":
        yo, so = oracle.integrate_batch(oracle.Model.mechanism("h2_lidryer"), y0, 0.0, 1e-5, 1e-6, 1e-10, rho=rho,
                                        fext_yc=F, group=group, threads=8, ls=oracle.LS_GMRES)
        end_state_check(yg, yo, 1e-6, 1e-10)
        assert abs(st["nli"] - so["nli"].sum()) <= 0.02 * so["nli"].sum()


def test_gmres_krylov_cap(oracle):
    """maxl = 2: many Newton failures (ncfn ~13 per cell), rounding-sensitive: the oracle's envelope."""
    y0, rho, F, prog = flame_field("drm19_class", 12, dt=1e-5)
    yg, sg, st, group = run_ls("drm19", y0, 1e-5, rho, F, "gmres", maxl=2)
    envelope_check(yg, sg, oracle, oracle.Model.mechanism("drm19_class"), y0, 1e-5, rho, F, ls=oracle.LS_GMRES,
                   maxl=2, group=group)


def test_linear_solver_unsupported_paths():
    b = P.Batch(64, 10, 1e-6, 1e-10)
    b.set_kernel("thread")
    b.set_model("h2")
    with pytest.raises(RuntimeError):
        b.set_linear_solver("gmres")
    b2 = P.Batch(64, 10, 1e-6, 1e-10)
    b2.set_model("h2")
    with pytest.raises(RuntimeError):
        b2.set_linear_solver("gmres", maxl=9)
    b2.set_jacobian("dq")
    with pytest.raises(RuntimeError):
        b2.set_linear_solver("diag")


# ------------------------------------------------------------------ explicit ERK (row f4)
def run_erk(name, y0, dt, rho, F, mxstep=100000):
    mech, n = MECH[name]
    b = P.Batch(y0.shape[1], n, 1e-6, 1e-10, mxstep=mxstep)
    b.set_model(name)
    b.set_method("erk4")
    cs = b.attach_cell_stats()
    y = cu(y0)
    b.integrate(0.0, dt, y, f_ext=cu(F), aux=cu(rho))
    return y.cpu().numpy(), {k: v.cpu().numpy() for k, v in cs.items()}, b.stats()


@pytest.mark.parametrize("name,dt", [("h2", 1e-7), ("h2", 1e-6), ("drm19", 1e-7), ("drm19", 1e-6)])
def test_erk_parity(oracle, name, dt):
    """GPU ERK (csrc/erk.cu) vs the oracle's orc_integrate_erk on 512 flame cells (every 8th of 16^3)."""
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 16, dt=dt)
    sel = np.arange(0, y0.shape[1], 8)
    y0, rho, F = np.ascontiguousarray(y0[:, sel]), rho[sel].copy(), np.ascontiguousarray(F[:, sel])
    yg, sg, st = run_erk(name, y0, dt, rho, F)
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F,
                                    threads=16, method=oracle.METHOD_ERK4, mxstep=100000)
    assert st["n_failed"] == 0 and np.array_equal(sg["status"], so["status"])
    end_state_check(yg, yo, 1e-6, 1e-10)
    same = np.mean([all(sg[k][c] == so[k][c] for k in ("nst", "nfe", "netf", "ncfn")) for c in range(len(sel))])
    print(f"{name} dt={dt} erk4: identical per-cell stats {same:.4f}; steps {st['nst']} rhs {st['nfe']}")
    assert same > 0.95
    assert st["nje"] == 0 and st["nni"] == 0 and np.all(sg["q_last"] == 4)


def test_erk_vs_bdf_direction(oracle):
    """P:426 (SPEC AC4): on the same GPU and cells the explicit method takes >= 10x the BDF steps at dt 1e-5."""
    y0, rho, F, prog = flame_field("h2_lidryer", 16, dt=1e-5)
    sel = np.where(prog > 0.02)[0][:256]
    y0, rho, F = np.ascontiguousarray(y0[:, sel]), rho[sel].copy(), np.ascontiguousarray(F[:, sel])
    ye, se, ste = run_erk("h2", y0, 1e-5, rho, F)
    b = P.Batch(len(sel), 10, 1e-6, 1e-10)
    b.set_model("h2")
    y = cu(y0)
    b.integrate(0.0, 1e-5, y, f_ext=cu(F), aux=cu(rho))
    stb = b.stats()
    assert ste["n_failed"] == 0 and stb["n_failed"] == 0
    assert ste["nst"] >= 10 * stb["nst"]
    assert 5.0 <= ste["nfe"] / ste["nst"] <= 6.5
    assert np.all(np.abs(ye - y.cpu().numpy()) <= 100 * (1e-6 * np.abs(ye) + 1e-10))


def test_erk_edge_cases():
    """NaN input -> NONFINITE (cell untouched); mxstep -> TOO_MUCH_WORK; ERK needs a mechanism model."""
    y0, rho, F, prog = flame_field("h2_lidryer", 4, dt=1e-6)
    y0 = np.ascontiguousarray(y0[:, :40])
    rho, F = rho[:40].copy(), np.ascontiguousarray(F[:, :40])
    y0[3, 5] = np.nan
    yg, sg, st = run_erk("h2", y0, 1e-6, rho, F, mxstep=3)
    assert sg["status"][5] == 5 and np.isnan(yg[3, 5])
    assert np.all((sg["status"] == 1) | (sg["status"] == 0) | (np.arange(40) == 5))
    b = P.Batch(8, 3, 1e-6, 1e-10)
    b.set_model("robertson")
    with pytest.raises(RuntimeError):
        b.set_method("erk4")


# ------------------------------------------------------------------ C5 mechanism per cell (n = 54)
@pytest.mark.parametrize("ls", ["dense", "gmres"])
def test_gri53_per_cell_parity(oracle, ls):
    """The 53-species GRI-3.0-class mechanism (config C5's, n = 54) per cell with the SPLIT kernel: the
    generated thread-per-cell RHS, the lanes Jacobian (K_jac, one cell per warp) and the register-row LU (K_lu,
    split_big.cuh) or GMRES; 512 flame cells at C5's dt_CFD = 1e-6 s vs the oracle, 10 tol on every cell."""
    y0, rho, F, prog = flame_field("gri53_class", 8, dt=1e-6)
    b = P.Batch(y0.shape[1], 54, 1e-6, 1e-10)
    b.set_model("gri53")
    if ls != "dense":
        b.set_linear_solver(ls)
    cs = b.attach_cell_stats()
    y = cu(y0)
    b.integrate(0.0, 1e-6, y, f_ext=cu(F), aux=cu(rho))
    st = b.stats()
    sg = {k: v.cpu().numpy() for k, v in cs.items()}
    yo, so = oracle.integrate_batch(oracle.Model.mechanism("gri53_class"), y0, 0.0, 1e-6, 1e-6, 1e-10, rho=rho,
                                    fext_yc=F, group=b.wrms_group, threads=16,
                                    ls=oracle.LS_DENSE if ls == "dense" else oracle.LS_GMRES)
    assert st["n_failed"] == 0 and np.array_equal(sg["status"], so["status"])
    end_state_check(y.cpu().numpy(), yo, 1e-6, 1e-10)
    same = np.mean([all(sg[k][c] == so[k][c] for k in STAT_KEYS) for c in range(y0.shape[1])])
    print(f"gri53 per cell {ls}: identical per-cell stats {same:.4f}; {st}")
    assert same > 0.9


def test_gri53_split_lu_parity(oracle):
    """K_lu for n = 54 (register rows, split_big.cuh) through a full integration whose every Newton solve uses
    it; plus the slot-reuse invariance with 64 slots for 512 cells (bit-identical)."""
    import os
    y0, rho, F, prog = flame_field("gri53_class", 8, dt=1e-6)

    def run():
        b = P.Batch(y0.shape[1], 54, 1e-6, 1e-10)
        b.set_model("gri53")
        y = cu(y0)
        b.integrate(0.0, 1e-6, y, f_ext=cu(F), aux=cu(rho))
        return y.cpu().numpy(), b.stats()

    y1, s1 = run()
    os.environ["BDFB_SPLIT_SLOTS"] = "64"
    try:
        y2, s2 = run()
    finally:
        del os.environ["BDFB_SPLIT_SLOTS"]
    assert np.array_equal(y1, y2) and s1 == s2


def test_gri53_erk_parity(oracle):
    y0, rho, F, prog = flame_field("gri53_class", 8, dt=1e-7)
    sel = np.arange(0, y0.shape[1], 4)
    y0, rho, F = np.ascontiguousarray(y0[:, sel]), rho[sel].copy(), np.ascontiguousarray(F[:, sel])
    b = P.Batch(len(sel), 54, 1e-6, 1e-10, mxstep=100000)
    b.set_model("gri53")
    b.set_method("erk4")
    cs = b.attach_cell_stats()
    y = cu(y0)
    b.integrate(0.0, 1e-7, y, f_ext=cu(F), aux=cu(rho))
    yo, so = oracle.integrate_batch(oracle.Model.mechanism("gri53_class"), y0, 0.0, 1e-7, 1e-6, 1e-10, rho=rho,
                                    fext_yc=F, threads=16, method=oracle.METHOD_ERK4, mxstep=100000)
    assert b.stats()["n_failed"] == 0
    end_state_check(y.cpu().numpy(), yo, 1e-6, 1e-10)
