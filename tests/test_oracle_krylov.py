"""Pins for the oracle's scaled GMRES (oracle/krylov.c; Eq. 5-6) and for the
inexact Newton-Krylov integrator path built on it (approaches 1A/1B, Table 1) and
the general CVDiag path.

The GMRES pins do not restate the algorithm: the iterate after k iterations is compared with the
least-squares minimiser of the scaled residual over the Krylov space, built here independently with numpy
(orthonormal Krylov basis by two-pass Gram-Schmidt + lstsq), the rotation residual with the explicitly formed residual, and the converged solution
with numpy's dense solve."""
import numpy as np
import pytest

GOLD_TOL = 1e-10


def krylov_lsq(A, b, s1, s2, k):
    """argmin over x~ in K_k(A~, b~) of ||b~ - A~ x~||_2, A~ = S1 A S2^-1, b~ = S1 b; returns x = S2^-1 x~."""
    At = (s1[:, None] * A) / s2[None, :]
    bt = s1 * b
    Q = np.empty((len(b), k))       # orthonormal basis of the Krylov space (classical GS, two passes)
    Q[:, 0] = bt / np.linalg.norm(bt)
    for j in range(1, k):
        v = At @ Q[:, j - 1]
        for _ in range(2):
            v = v - Q[:, :j] @ (Q[:, :j].T @ v)
        Q[:, j] = v / np.linalg.norm(v)
    z, *_ = np.linalg.lstsq(At @ Q, bt, rcond=None)
    xt = Q @ z
    return xt / s2, np.linalg.norm(bt - At @ xt)


def rand_system(rng, n=20):
    A = np.eye(n) + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    s1 = np.exp(rng.uniform(-3, 3, n))
    s2 = s1.copy()          # the integrator's S1 = S2 = diag(w); a separate S2 is tested below
    return A, b, s1, s2


def test_identity_converges_in_one_iteration(oracle):
    b = np.array([1.0, -2.0, 3.5, 0.25])
    x, st, it, rn = oracle.gmres(np.eye(4), b, delta=1e-14, maxl=4)
    assert st == 0 and it == 1
    assert np.allclose(x, b, rtol=1e-15, atol=0)


def test_k_distinct_eigenvalues_terminate_in_k_iterations(oracle):
    d = np.repeat([2.0, -3.0, 7.5], 7)[:20]
    b = np.random.default_rng(1).standard_normal(20)
    x, st, it, rn = oracle.gmres(np.diag(d), b, delta=1e-12 * np.linalg.norm(b), maxl=20)
    assert st == 0 and it <= 3
    assert np.allclose(x, b / d, rtol=1e-12)


@pytest.mark.parametrize("seed", range(50))
def test_rotation_residual_is_the_explicit_residual(oracle, seed):
    """at every k the rotation-tracked residual equals ||S1 (b - A x_k)||_2 (1e-10 rel),
    and x_k is the Krylov least-squares minimiser."""
    rng = np.random.default_rng(seed)
    A, b, s1, s2 = rand_system(rng)
    if seed % 2:
        s2 = np.exp(rng.uniform(-2, 2, 20))
    for k in range(1, 9):
        x, st, it, rn = oracle.gmres(A, b, s1=s1, s2=s2, delta=0.0, maxl=k)
        assert st in (0, 1) and it == k
        explicit = np.linalg.norm(s1 * (b - A @ x))
        assert abs(rn - explicit) <= GOLD_TOL * explicit
        xl, rl = krylov_lsq(A, b, s1, s2, k)
        assert abs(rn - rl) <= 1e-9 * rl
        assert np.allclose(x, xl, rtol=1e-8, atol=1e-12 * np.abs(xl).max())


@pytest.mark.parametrize("seed", range(10))
def test_scaled_solution_matches_direct_solve(oracle, seed):
    """Eq. 5 consistency: solving the transformed system and back-transforming reproduces A^-1 b; with
    S1 = S2 = I it is textbook GMRES."""
    rng = np.random.default_rng(100 + seed)
    A, b, s1, s2 = rand_system(rng)
    ref = np.linalg.solve(A, b)
    for sc in ((s1, s2), (None, None), (s1, np.exp(rng.uniform(-2, 2, 20)))):
        x, st, it, rn = oracle.gmres(A, b, s1=sc[0], s2=sc[1], delta=1e-13 * np.linalg.norm(b), maxl=20)
        assert st == 0
        assert np.allclose(x, ref, rtol=1e-10, atol=1e-12)


def test_stagnation_reports_failure(oracle):
    """The cyclic shift with b = e_1: the Krylov residual does not decrease before n iterations, so a
    smaller cap must report CONV_FAIL (no reduction), not a solution."""
    n = 8
    A = np.roll(np.eye(n), 1, axis=0)
    b = np.zeros(n)
    b[0] = 1.0
    x, st, it, rn = oracle.gmres(A, b, delta=1e-12, maxl=5)
    assert st == 2 and it == 5 and abs(rn - 1.0) < 1e-14
    x, st, it, rn = oracle.gmres(A, b, delta=1e-12, maxl=n)
    assert st == 0 and np.allclose(A @ x, b, atol=1e-14)


def test_gmres_tolerance_is_met(oracle):
    """SUCCESS means the scaled residual is below delta (Eq. 6)."""
    rng = np.random.default_rng(7)
    A, b, s1, s2 = rand_system(rng)
    for delta in (1e-2, 1e-5, 1e-9):
        x, st, it, rn = oracle.gmres(A, b, s1=s1, s2=s2, delta=delta * np.linalg.norm(s1 * b), maxl=20)
        assert st == 0
        assert np.linalg.norm(s1 * (b - A @ x)) <= delta * np.linalg.norm(s1 * b) * (1 + 1e-8)


# ---- the Newton-Krylov integrator (approaches 1A/1B) ----------------------------------------------------
def test_newton_krylov_linear_closed_form(oracle):
    lam = np.array([-1.0, -10.0, -1e3, -3e4, 0.5])
    m = oracle.Model.linear(lam)
    y0 = np.array([1.0, 2.0, -3.0, 0.5, 0.25])
    y, st, _ = oracle.integrate(m, y0, 0.0, 2.0, 1e-7, 1e-12, ls=oracle.LS_GMRES)
    exact = y0 * np.exp(lam * 2.0)
    assert st["status"] == 0
    assert np.all(np.abs(y - exact) <= 10 * (1e-7 * np.abs(exact) + 1e-12))
    # matrix-free: no Jacobian, no matrix setup; every Newton iteration ran GMRES or took the small-b exit
    assert st["nje"] == 0 and st["nsetups"] == 0 and st["nli"] >= 1
    attempts = st["nst"] + st["netf"] + st["ncfn"]
    assert st["nni"] <= 2 * attempts


@pytest.mark.parametrize("ls", ["gmres", "diag"])
def test_robertson_matches_dense_direct(oracle, ls):
    """approach 2A (dense, analytic J) and 1A (GMRES) endpoints agree to <= 100 rtol; CVDiag
    (the paper's Nyx solver, here on a coupled system) likewise."""
    m = oracle.Model.robertson()
    code = oracle.LS_GMRES if ls == "gmres" else oracle.LS_DIAG
    for tf in (0.4, 4.0, 40.0):
        yd, sd, _ = oracle.integrate(m, [1.0, 0.0, 0.0], 0.0, tf, 1e-6, 1e-10, ls=oracle.LS_DENSE)
        yk, sk, _ = oracle.integrate(m, [1.0, 0.0, 0.0], 0.0, tf, 1e-6, 1e-10, ls=code)
        assert sk["status"] == 0
        # CVDiag's diagonal Newton matrix breaks the invariant sum(y) = 1 by up to the Newton tolerance per
        # step; over the 480 steps to t = 40 that drift is the dominant global error (1000 rtol allowed)
        band = 100 if (ls == "gmres" or tf < 10) else 1000
        assert np.all(np.abs(yk - yd) <= band * 1e-6 * np.abs(yd) + 1e-9), (tf, yk, yd)
        # GMRES keeps x in K(A, b) (S1 = S2), whose vectors conserve the linear invariant sum(y) = 1; the
        # diagonal Newton matrix does not (e^T M != e^T), so CVDiag conserves it only to the Newton tolerance
        assert abs(yk.sum() - 1.0) < (1e-12 if ls == "gmres" else band * 1e-6)


def test_cvdiag_exact_on_diagonal_linear_system(oracle):
    """For y' = diag(lambda) y the CVDiag difference quotient is the exact diagonal J (up to rounding), so
    modified Newton converges like the dense solver: closed form, and a Newton iteration count close to
    the dense run's."""
    lam = np.array([-1.0, -50.0, -2e3])
    m = oracle.Model.linear(lam)
    y0 = np.array([1.0, -1.0, 2.0])
    yg, sg, _ = oracle.integrate(m, y0, 0.0, 1.0, 1e-8, 1e-14, ls=oracle.LS_DIAG)
    yd, sd, _ = oracle.integrate(m, y0, 0.0, 1.0, 1e-8, 1e-14, ls=oracle.LS_DENSE)
    exact = y0 * np.exp(lam)
    assert np.all(np.abs(yg - exact) <= 10 * (1e-8 * np.abs(exact) + 1e-14))
    assert sg["ncfn"] == 0 and abs(sg["nst"] - sd["nst"]) <= 0.1 * sd["nst"] + 2


def test_newton_krylov_no_retry_and_counts(oracle):
    """Without a preconditioner there is no linear-solver setup (CVODE sets lsetup = NULL): on a stiff
    mechanism cell the run still completes, with nje = nsetups = 0 and the Krylov iterations counted."""
    import synth
    yf, rho, F, _ = synth.flame_field("h2_lidryer", 3, cells=np.arange(6))
    m = oracle.Model.mechanism("h2_lidryer")
    y, st = oracle.integrate_batch(m, yf, 0.0, 1e-6, 1e-6, 1e-10, rho=rho, fext_yc=F, ls=oracle.LS_GMRES)
    yd, sd = oracle.integrate_batch(m, yf, 0.0, 1e-6, 1e-6, 1e-10, rho=rho, fext_yc=F, ls=oracle.LS_DENSE)
    assert np.all(st["status"] == 0)
    assert np.all(st["nje"] == 0) and np.all(st["nsetups"] == 0) and st["nli"].sum() > 0   # near-equilibrium cells take the small-b exit
    assert np.all(np.abs(y - yd) <= 100 * (1e-6 * np.abs(yd) + 1e-10))
