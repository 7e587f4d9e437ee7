"""Pins for the oracle parts the round-1 review found unpinned (VERDICT r1 "weak #2"):

* the step/order controller (PREPARE_NEXT, cvChooseEta + cvSetEta; listing §8(c).2, readings R7/R8),
* the error-test coefficients tq[1] and tq[3] (order q-1 / q+1 estimates),
* the Newton iteration (replayed with numpy dense solves),
* the plain-arithmetic mode (libm pow, true division) against the R25/R16 mode,
* the KWH heating/cooling sum (density scaling of two-body cooling, the fully ionised limit),
* falloff (Lindemann / Troe limits) and forward Arrhenius rates on single-reaction toy mechanisms,
* the R19 parity scale orc_rhs_scale.

No check below restates the oracle's formula: each one uses a special value, a limit, an invariant, a
textbook constant or an independent computation (numpy, exact rationals)."""
import math
from fractions import Fraction

import numpy as np
import pytest

from synth import flame_field, robertson_field

ADDON = 1e-6


# ---------------------------------------------------------------- controller
def _bdf_err_const(k):
    """|C_{k+1}| of BDF-k: beta0 / (k+1), beta0 = 1 / sum_{j<=k} 1/j (Hairer-Wanner III.1)."""
    return Fraction(1, sum(Fraction(1, j) for j in range(1, k + 1))) / (k + 1)


@pytest.mark.parametrize("q", [1, 2, 3, 4, 5])
def test_tq1_tq3_constant_step_are_neighbour_order_error_constants(oracle, q):
    """At constant h: tq[1] = q! |C| of BDF-(q-1) (||zn[q]|| tq[1] is the order-(q-1) LTE, zn[q] = h^q y^(q)/q!)
    and tq[3] = |C| of BDF-(q+1) (the order-(q+1) estimate).  tq[1] = 1 at q = 1 by definition."""
    h = 0.37
    _, tq = oracle.set_bdf(q, h, [h] * 6, qwait=1)
    t1 = 1.0 if q == 1 else float(_bdf_err_const(q - 1) * math.factorial(q))
    assert tq[1] == pytest.approx(t1, rel=1e-13)
    assert tq[3] == pytest.approx(float(_bdf_err_const(q + 1)), rel=1e-13)


@pytest.mark.parametrize("plain", [False, True])
@pytest.mark.parametrize("q", [1, 2, 3, 4, 5])
def test_controller_special_values(oracle, q, plain):
    """eta_q = 1/((BIAS2 dsm)^(1/L) + ADDON): at dsm = (1/2 - ADDON)^L / 6, eta_q = 2 (BIAS2 = 6, exponent 1/L).
    eta_{q-1} (BIAS1 = 6, exponent 1/q) and eta_{q+1} (BIAS3 = 10, exponent 1/(L+1)) likewise, each winning
    against a large dsm (tiny eta_q).  Rounding of the root is the only slack."""
    L = q + 1
    x = 0.5 - ADDON
    # order kept: qwait != 0 -> only eta_q is formed
    eta, qp, hp, qw = oracle.choose_eta(q, 1, x ** L / 6.0, etamax=10.0, h=0.25, plain=plain)
    assert eta == pytest.approx(2.0, rel=1e-14) and qp == q and qw == 1 and hp == pytest.approx(0.5, rel=1e-14)
    big = 1e6   # eta_q ~ 0.02
    if q > 1:
        eta, qp, _, qw = oracle.choose_eta(q, 0, big, ddn=x ** q / 6.0, etamax=10.0, plain=plain)
        assert qp == q - 1 and eta == pytest.approx(2.0, rel=1e-14) and qw == 2
    if q < 5:
        eta, qp, _, _ = oracle.choose_eta(q, 0, big, ddn=big, dup=x ** (L + 1) / 10.0, etamax=10.0, plain=plain)
        assert qp == q + 1 and eta == pytest.approx(2.0, rel=1e-14)


def test_controller_threshold_caps_and_ties(oracle):
    """THRESH: eta < 1.5 keeps h; growth capped by etamax (first step 1e4, later 10); hmax caps h';
    after a failure (etamax = 1) h is kept and qwait >= 2; exact ties prefer q, then q-1, then q+1 (R8)."""
    def dsm_for(eta, L):
        return (1.0 / eta - ADDON) ** L / 6.0
    eta, qp, hp, _ = oracle.choose_eta(2, 1, dsm_for(1.4, 3), h=0.3)
    assert (eta, qp, hp) == (1.0, 2, 0.3)
    eta, _, hp, _ = oracle.choose_eta(2, 1, dsm_for(1.6, 3), h=0.3)
    assert eta == pytest.approx(1.6, rel=1e-13) and hp == pytest.approx(0.48, rel=1e-13)
    eta, _, _, _ = oracle.choose_eta(3, 1, 0.0, etamax=10.0)          # ||LTE|| -> 0: growth cap
    assert eta == 10.0
    eta, _, _, _ = oracle.choose_eta(1, 1, 1e-30, etamax=1e4)          # first step cap ETAMX1
    assert eta == 1e4
    eta, _, hp, _ = oracle.choose_eta(2, 1, 0.0, etamax=10.0, h=0.3, hmax=0.9)
    assert hp == pytest.approx(0.9, rel=1e-15) and eta == pytest.approx(3.0, rel=1e-15)
    eta, qp, hp, qw = oracle.choose_eta(3, 0, 1e-3, etamax=1.0, h=0.3)
    assert (eta, qp, hp, qw) == (1.0, 3, 0.3, 2)
    # exact three-way tie (all norms zero -> every eta = 1/ADDON): keep q
    _, qp, _, _ = oracle.choose_eta(3, 0, 0.0, ddn=0.0, dup=0.0, etamax=10.0)
    assert qp == 3
    # tie between q-1 and q+1 above eta_q: prefer q-1
    _, qp, _, _ = oracle.choose_eta(3, 0, 1e-6, ddn=0.0, dup=0.0, etamax=10.0)
    assert qp == 2
    # q+1 wins only when strictly larger
    _, qp, _, _ = oracle.choose_eta(3, 0, 1e-6, ddn=1e-6, dup=0.0, etamax=10.0)
    assert qp == 4


def test_eta_scales_with_the_order_of_the_error(oracle):
    """Asymptotically eta_q ~ (6 dsm)^(-1/L): multiplying dsm by 2^L halves eta (the LTE is O(h^L))."""
    for q in range(1, 6):
        L = q + 1
        e1, *_ = oracle.choose_eta(q, 1, 1e-4, etamax=1e30)
        e2, *_ = oracle.choose_eta(q, 1, 1e-4 * 2.0 ** L, etamax=1e30)
        assert e1 / e2 == pytest.approx(2.0, rel=1e-4)


# ---------------------------------------------------------------- Newton replay
def _newton_replay(oracle, model, zn0, zn1, ewt, h, rl1, tol, rho, fext):
    """The listing's NEWTON (forced setup, J at zn0, gamrat = 1, R = 1) with numpy dense solves and a plain
    sequential WRMS; returns (acor, iterations, rhs evaluations)."""
    n = len(zn0)
    gamma = h * rl1
    J, r = oracle.jac(model, zn0, rho, fext)
    assert r == 0
    M = np.eye(n) - gamma * J
    wrms = lambda v: math.sqrt(math.fsum((v * ewt) ** 2) / n)
    ycor = np.zeros(n)
    crate, dprev, nfe = 1.0, 0.0, 0
    for m in range(3):
        f, r = oracle.rhs(model, zn0 + ycor, rho, fext)
        nfe += 1
        G = ycor + rl1 * zn1 - gamma * f
        d = np.linalg.solve(M, -G)
        ycor = ycor + d
        dn = wrms(d)
        if m > 0:
            crate = max(0.3 * crate, dn / dprev)
        if dn * min(1.0, crate) <= tol:
            return ycor, m + 1, nfe
        if m >= 1 and dn > 2.0 * dprev:
            return None, m + 1, nfe
        dprev = dn
    return None, 3, nfe


@pytest.mark.parametrize("name", ["h2_lidryer", "drm19_class"])
def test_newton_iterates_match_numpy_replay(oracle, name):
    """Newton iterates vs an independent numpy dense-solve replay on predicted flame states: same
    iteration count and RHS count, corrections equal to ~1e-10 of their WRMS size."""
    m = oracle.Model.mechanism(name)
    y, rho, F, prog = flame_field(name, 6, cells=np.arange(40))
    rng = np.random.default_rng(7)
    checked = 0
    for c in range(y.shape[1]):
        zn0 = y[:, c].copy()
        f0, _ = oracle.rhs(m, zn0, rho[c], F[:, c])
        ewt = 1.0 / (1e-6 * np.abs(zn0) + 1e-10)
        h = 10.0 ** rng.uniform(-9, -6)
        q = int(rng.integers(1, 6))
        l, tq = oracle.set_bdf(q, h, [h] * 6, qwait=2)
        rl1 = 1.0 / l[1]
        # predicted state: a step along f0 perturbed, so the corrector has work to do
        zn1 = h * f0 * (1.0 + 0.05 * rng.standard_normal(len(zn0)))
        st, acor, acnrm, nni, nfe = oracle.newton_once(m, zn0, zn1, ewt, h, rl1, tq[4], rho=rho[c], fext=F[:, c])
        ref, its, nfe_ref = _newton_replay(oracle, m, zn0, zn1, ewt, h, rl1, tq[4], rho[c], F[:, c])
        if ref is None:
            assert st != 0
            continue
        assert st == 0 and nni == its and nfe == nfe_ref
        scale = math.sqrt(np.mean((ref * ewt) ** 2))
        assert np.max(np.abs((acor - ref) * ewt)) <= 1e-9 * max(scale, 1e-300) + 1e-12
        checked += 1
    assert checked >= 30


def test_newton_linear_problem_first_correction_exact(oracle):
    """On f = lambda y the first Newton correction solves the linear system exactly: acor equals the closed form
    (I - gamma Lambda)^{-1} (gamma lambda zn0 - rl1 zn1)."""
    lam = np.array([-3.0, -1e3, 2.0, -0.5])
    m = oracle.Model.linear(lam)
    zn0 = np.array([1.0, 0.5, -2.0, 3.0])
    zn1 = np.array([0.01, -0.2, 0.03, 0.0])
    h, rl1 = 1e-2, 1.0
    ewt = 1.0 / (1e-6 * np.abs(zn0) + 1e-10)
    st, acor, _, nni, _ = oracle.newton_once(m, zn0, zn1, ewt, h, rl1, 1e-30 + 0.05)
    g = h * rl1
    exact = (g * lam * zn0 - rl1 * zn1) / (1.0 - g * lam)
    assert st == 0 and nni <= 2
    np.testing.assert_allclose(acor, exact, rtol=1e-13, atol=1e-16)


# ---------------------------------------------------------------- plain mode
def test_lu_solve_plain_division_matches_exact_rational(oracle):
    """Plain LU_SOLVE (true division) reproduces an exact-rational substitution on the same factors, rounded
    step by step as the listing orders it (independent Python code)."""
    rng = np.random.default_rng(11)
    for n in (1, 3, 7, 22):
        A = rng.standard_normal((n, n)) + n * np.eye(n)
        LU, piv, info = oracle.lu_factor(A)
        assert info == 0
        b = rng.standard_normal(n)
        x = oracle.lu_solve(LU, piv, b, plain=True)
        y = [float(v) for v in b]
        for k in range(n):
            p = int(piv[k])
            y[k], y[p] = y[p], y[k]
        fma = lambda a, bb, c: float(Fraction(a) * Fraction(bb) + Fraction(c))
        for k in range(n - 1):
            for i in range(k + 1, n):
                y[i] = fma(-LU[i, k], y[k], y[i])
        for k in range(n - 1, 0, -1):
            y[k] = float(Fraction(y[k]) / Fraction(float(LU[k, k])))
            for i in range(k):
                y[i] = fma(-LU[i, k], y[k], y[i])
        y[0] = float(Fraction(y[0]) / Fraction(float(LU[0, 0])))
        assert np.array_equal(x, np.array(y))
        # and R16 (reciprocal multiply) differs from it by at most a few ulp
        x16 = oracle.lu_solve(LU, piv, b)
        np.testing.assert_allclose(x16, x, rtol=64 * n * 2.0 ** -52, atol=1e-300)


@pytest.mark.parametrize("name,dt", [("robertson", 40.0), ("h2_lidryer", 1e-5), ("drm19_class", 1e-5)])
def test_plain_mode_end_states_within_band_of_r25_mode(oracle, name, dt):
    """The plain-arithmetic oracle (libm pow roots, true division) and the R25/R16 oracle agree within the
    end-state band |dy| <= 10 (rtol |y| + atol) on every cell; nearly all cells take identical decisions."""
    if name == "robertson":
        m = oracle.Model.robertson()
        y0 = robertson_field(64)
        rho = F = None
    else:
        m = oracle.Model.mechanism(name)
        y0, rho, F, _ = flame_field(name, 6 if name == "drm19_class" else 5, cells=np.arange(0, 4096, 64))
    yp, sp = oracle.integrate_batch(m, y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F, plain=True, threads=4)
    yr, sr = oracle.integrate_batch(m, y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F, threads=4)
    assert np.all(sp["status"] == 0) and np.all(sr["status"] == 0)
    tol = 10.0 * (1e-6 * np.abs(yp) + 1e-10)
    assert np.all(np.abs(yr - yp) <= tol)
    same = np.mean((sp["nst"] == sr["nst"]) & (sp["nfe"] == sr["nfe"]) & (sp["netf"] == sr["netf"]))
    assert same >= 0.9


# ---------------------------------------------------------------- KWH (Nyx) RHS
def _kwh(oracle, **kw):
    return oracle.Model.nyx_kwh(**kw)


def test_kwh_two_body_cooling_scales_with_density(oracle):
    """Without photo-ionisation, photo-heating and Compton cooling ((1+z)^4 = 0 at z = -1) every process is
    two-body (rate per volume ~ n^2), so R(e) = -Lambda/rho is exactly proportional to rho at fixed e."""
    m = _kwh(oracle, z=-1.0, gph=(0.0, 0.0, 0.0), eph=(0.0, 0.0, 0.0))
    for T in (2e4, 1e5, 3e5, 1e6, 1e7):
        e = 1.5 * 1.380649e-16 * T / (0.59 * 1.67262192369e-24)
        f1, r1 = oracle.rhs(m, [e], rho=1e-27)
        f2, r2 = oracle.rhs(m, [e], rho=4e-27)
        assert r1 == 0 and r2 == 0 and f1[0] < 0.0
        assert f2[0] == pytest.approx(4.0 * f1[0], rel=1e-9)


def test_kwh_fully_ionised_limit_is_free_free_plus_compton(oracle):
    """T >~ 1e7 K: hydrogen and helium fully ionised and the cooling tends to thermal bremsstrahlung
    Lambda_ff = 1.42e-27 g_ff T^(1/2) n_e sum Z^2 n_i (Gaunt factor 1.1 <= g_ff <= 1.5) plus inverse Compton
    Lambda_C = 5.41e-36 n_e T (1+z)^4 (Ikeuchi & Ostriker; KWH96) -- recombination and collisional terms are a
    few per cent at most.  Photo terms off."""
    z = 3.0
    m = _kwh(oracle, z=z, gph=(0.0, 0.0, 0.0), eph=(0.0, 0.0, 0.0))
    rho = 1e-27
    for T in (3e7, 1e8):
        e = 1.5 * 1.380649e-16 * T / (0.59 * 1.67262192369e-24)
        st, r = oracle.kwh_state(m, e, rho)
        assert r == 0
        nH = 0.76 * rho / 1.67262192369e-24
        nHe = nH * 0.24 / (4 * 0.76)
        assert st["nHp"] == pytest.approx(nH, rel=1e-3) and st["nHepp"] == pytest.approx(nHe, rel=1e-3)
        ne, TT = st["ne"], st["T"]
        ff = lambda g: 1.42e-27 * g * math.sqrt(TT) * ne * (st["nHp"] + st["nHep"] + 4.0 * st["nHepp"])
        comp = 5.41e-36 * ne * TT * (1.0 + z) ** 4
        f, rr = oracle.rhs(m, [e], rho=rho)
        lam = -f[0] * rho
        assert ff(1.1) + comp <= lam <= 1.05 * (ff(1.5) + comp)


# ---------------------------------------------------------------- falloff / Arrhenius on toy mechanisms
def _toy(rx):
    nasa = {"Tmid": 1000.0, "low": [3.5, 0, 0, 0, 0, -1000.0, 3.0], "high": [3.5, 0, 0, 0, 0, -1000.0, 3.0]}
    sp = [{"name": n, "composition": {"N": 2}, "W": 28.0, "nasa": nasa} for n in ("A", "B", "N2")]
    return {"name": "toy", "species": sp, "reactions": [rx]}


def _rate(oracle, table, T, rho, yA=0.2):
    """k of A -> B (irreversible) from the oracle RHS: f_A = W_A wdot_A / rho = -k(rho) Y_A."""
    md = oracle.MechData(table)
    m = oracle.Model("toy", n=md.K + 1, mech=md)
    y = np.array([yA, 0.0, 1.0 - yA, T])
    f, r = oracle.rhs(m, y, rho=rho)
    assert r == 0
    return -f[0] / yA


EFF = {"A": 1.0, "B": 1.0, "N2": 1.0}
MOLAR = 1.0 / 28.0     # [M] = rho * sum eff Y / W = rho / 28


def test_arrhenius_forward_rate(oracle):
    """k = A T^b exp(-Ea/(R_c T)), R_c = 1.98720 cal/mol/K: the activation energy from two temperatures and the
    temperature exponent at Ea = 0."""
    rx = {"equation": "A => B", "reactants": ["A"], "products": ["B"], "reversible": False, "type": "elementary",
          "A": 3.0e9, "b": 0.0, "Ea": 20000.0}
    k1, k2 = _rate(oracle, _toy(rx), 1000.0, 1e-3), _rate(oracle, _toy(rx), 1500.0, 1e-3)
    assert k2 / k1 == pytest.approx(math.exp(-20000.0 / 1.98720425864083 * (1 / 1500.0 - 1 / 1000.0)), rel=1e-12)
    assert k1 == pytest.approx(3.0e9 * math.exp(-20000.0 / (1.98720425864083 * 1000.0)), rel=1e-12)
    rx2 = dict(rx, b=1.7, Ea=0.0)
    assert _rate(oracle, _toy(rx2), 1600.0, 1e-3) / _rate(oracle, _toy(rx2), 800.0, 1e-3) == pytest.approx(2 ** 1.7,
                                                                                                          rel=1e-12)


def test_three_body_rate_is_linear_in_M(oracle):
    rx = {"equation": "A + M => B + M", "reactants": ["A"], "products": ["B"], "reversible": False,
          "type": "three_body", "A": 1e12, "b": 0.0, "Ea": 0.0, "efficiencies": EFF}
    k1, k2 = _rate(oracle, _toy(rx), 1200.0, 1e-4), _rate(oracle, _toy(rx), 1200.0, 3e-4)
    assert k2 == pytest.approx(3.0 * k1, rel=1e-13)
    assert k1 == pytest.approx(1e12 * 1e-4 * MOLAR, rel=1e-13)


def _falloff_rx(kind):
    rx = {"equation": "A (+M) => B (+M)", "reactants": ["A"], "products": ["B"], "reversible": False,
          "type": "lindemann", "A": 5e9, "b": 0.3, "Ea": 5000.0, "efficiencies": EFF,
          "low": {"A": 3e16, "b": -1.0, "Ea": 2000.0}}
    if kind == "troe":
        rx = dict(rx, type="troe", troe=[0.6, 200.0, 1500.0, 4000.0])
    elif kind == "troe_fc1":
        rx = dict(rx, type="troe", troe=[1.0, 1e-30, 1e300])
    return rx


def _k_arr(A, b, Ea, T):
    return A * T ** b * math.exp(-Ea / (1.98720425864083 * T))


def test_lindemann_pressure_limits(oracle):
    """Lindemann k = k_inf Pr/(1+Pr), Pr = k0 [M]/k_inf: low pressure -> k0 [M], high pressure -> k_inf."""
    T = 1300.0
    rx = _falloff_rx("lindemann")
    kinf, k0 = _k_arr(5e9, 0.3, 5000.0, T), _k_arr(3e16, -1.0, 2000.0, T)
    klo = _rate(oracle, _toy(rx), T, 1e-14)
    khi = _rate(oracle, _toy(rx), T, 1e8)
    assert klo / (k0 * 1e-14 * MOLAR) == pytest.approx(1.0, rel=1e-9)
    assert khi / kinf == pytest.approx(1.0, rel=1e-8)


def test_troe_with_unit_fcent_is_lindemann(oracle):
    """Troe with F_cent = 1 (a = 1, T1 -> inf, T3 -> 0, no T2: F_cent = (1-a) e^(-T/T3) + a e^(-T/T1) = 1) has
    log F = 0 at every pressure, i.e. it is Lindemann."""
    T = 1300.0
    tr, li = _falloff_rx("troe_fc1"), _falloff_rx("lindemann")
    for rho in (1e-10, 1e-6, 1e-4, 1e-2, 1.0, 1e4):
        assert _rate(oracle, _toy(tr), T, rho) == pytest.approx(_rate(oracle, _toy(li), T, rho), rel=1e-12)


@pytest.mark.parametrize("T", [900.0, 1300.0, 2100.0])
def test_troe_centre_of_falloff(oracle, T):
    """At the centre of the falloff curve, log10 Pr = -c = 0.4 + 0.67 log10 F_cent, Troe's broadening factor is
    exactly F = F_cent (Troe 1983): k = k_inf (Pr/(1+Pr)) F_cent, with
    F_cent = (1-a) e^(-T/T***) + a e^(-T/T*) + e^(-T**/T)."""
    rx = _falloff_rx("troe")
    kinf, k0 = _k_arr(5e9, 0.3, 5000.0, T), _k_arr(3e16, -1.0, 2000.0, T)
    a, T3, T1, T2 = rx["troe"]
    Fc = (1 - a) * math.exp(-T / T3) + a * math.exp(-T / T1) + math.exp(-T2 / T)
    Pr = 10.0 ** (0.4 + 0.67 * math.log10(Fc))
    rho = Pr * kinf / (k0 * MOLAR)
    k = _rate(oracle, _toy(rx), T, rho)
    assert k == pytest.approx(kinf * Pr / (1.0 + Pr) * Fc, rel=1e-9)


# ---------------------------------------------------------------- R19 scale
@pytest.mark.parametrize("name", ["h2_lidryer", "drm19_class"])
def test_rhs_scale_bounds_the_rhs(oracle, name):
    """S_i >= |f_i - F_i| (triangle inequality over the same terms) on flame states; S = |f| exactly when the
    RHS has a single term (one irreversible reaction, no forcing)."""
    m = oracle.Model.mechanism(name)
    y, rho, F, _ = flame_field(name, 6, cells=np.arange(0, 4096, 97))
    for c in range(y.shape[1]):
        f, r = oracle.rhs(m, y[:, c], rho[c])
        S, r2 = oracle.rhs_scale(m, y[:, c], rho[c])
        assert r == 0 and r2 == 0
        assert np.all(S >= np.abs(f) * (1 - 1e-12))
    rx = {"equation": "A => B", "reactants": ["A"], "products": ["B"], "reversible": False, "type": "elementary",
          "A": 3.0e9, "b": 0.0, "Ea": 20000.0}
    md = oracle.MechData(_toy(rx))
    mt = oracle.Model("toy", n=md.K + 1, mech=md)
    yt = np.array([0.2, 0.1, 0.7, 1200.0])
    f, _ = oracle.rhs(mt, yt, rho=1e-3)
    S, _ = oracle.rhs_scale(mt, yt, rho=1e-3)
    np.testing.assert_allclose(S[:2], np.abs(f[:2]), rtol=1e-14)
