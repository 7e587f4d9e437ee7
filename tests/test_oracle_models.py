"""Pins for the oracle's model right-hand sides.

Constant-volume reactor: complex-step J equals central differences of the RHS;
mass, element and internal-energy conservation (u_k from the NASA-7 data,
not from the oracle); thermodynamic equilibrium (sum nu mu = 0 per reaction)
reached by long integration pins the Kc convention.  KWH: collisional and
photo-ionisation equilibrium relations (KWH96 eqs. 33-38) hold at the
regula-falsi root, written here from the published Appendix-B rate table."""
import math

import numpy as np
import pytest

RU = 8.31446261815324e7
PATM = 1013250.0
MECHS = {"h2_lidryer": ({"H2": 0.02852, "O2": 0.22635, "N2": 0.74513}, 1100.0),
         "drm19_class": ({"CH4": 0.05519, "O2": 0.22015, "N2": 0.72466}, 1400.0),
         "gri53_class": ({"CH4": 0.05519, "O2": 0.22015, "N2": 0.72466}, 1400.0)}   # C5 (n = 54)


def nasa(table, T):
    cp, h, s = [], [], []
    for sp in table["species"]:
        a = sp["nasa"]["low"] if T < sp["nasa"]["Tmid"] else sp["nasa"]["high"]
        cp.append(a[0] + a[1] * T + a[2] * T**2 + a[3] * T**3 + a[4] * T**4)
        h.append(a[0] + a[1] * T / 2 + a[2] * T**2 / 3 + a[3] * T**3 / 4 + a[4] * T**4 / 5 + a[5] / T)
        s.append(a[0] * math.log(T) + a[1] * T + a[2] * T**2 / 2 + a[3] * T**3 / 3 + a[4] * T**4 / 4 + a[6])
    return np.array(cp), np.array(h), np.array(s)


def initial_state(m, name):
    fr, T0 = MECHS[name]
    Y = np.zeros(m.mech.K)
    for k, v in fr.items():
        Y[m.mech.species.index(k)] = v
    Y /= Y.sum()
    rho = PATM / (RU * T0 * np.sum(Y / m.mech.W))
    return np.concatenate([Y, [T0]]), rho


def reacting_states(oracle, m, name, count=6):
    y0, rho = initial_state(m, name)
    out, y, t = [], y0.copy(), 0.0
    for tt in np.logspace(-6, -1.5, 60):
        y, st, _ = oracle.integrate(m, y, t, tt, 1e-9, 1e-16, rho)
        t = tt
        if y[-1] > y0[-1] + 50 and len(out) < count:
            out.append(y.copy())
    return out, rho


@pytest.mark.parametrize("name", list(MECHS))
def test_mech_jacobian_is_derivative_of_rhs(oracle, name):
    m = oracle.Model.mechanism(name)
    states, rho = reacting_states(oracle, m, name)
    assert states
    for y in states[:3]:
        J, r = oracle.jac(m, y, rho)
        assert r == 0
        for j in range(m.n):
            h = 1e-5 * max(abs(y[j]), 1e-7 if j < m.n - 1 else 1.0)
            e = np.zeros(m.n)
            e[j] = h
            fd = (oracle.rhs(m, y + e, rho)[0] - oracle.rhs(m, y - e, rho)[0]) / (2 * h)
            scale = np.abs(J).max(axis=1) + 1e-300
            assert np.all(np.abs(J[:, j] - fd) <= 1e-5 * scale), (name, j)


@pytest.mark.parametrize("name", list(MECHS))
def test_mech_conservation_mass_elements_energy(oracle, name):
    m = oracle.Model.mechanism(name)
    table = m.mech.table
    states, rho = reacting_states(oracle, m, name)
    elems = sorted({e for sp in table["species"] for e in sp["composition"]})
    E = np.array([[sp["composition"].get(e, 0) for sp in table["species"]] for e in elems], dtype=float)
    W = m.mech.W
    for y in states:
        f, r = oracle.rhs(m, y, rho)
        fy, fT = f[:-1], f[-1]
        scale = np.abs(fy).sum() + 1e-300
        assert abs(fy.sum()) <= 1e-12 * scale                      # sum_k dY_k/dt = 0
        assert np.all(np.abs(E @ (fy / W)) <= 1e-12 * (E @ (np.abs(fy) / W) + 1e-300))
        T = y[-1]
        cp, h, _ = nasa(table, T)
        u = (h - 1.0) * RU * T / W                                   # erg/g
        cv = np.sum(y[:-1] * (cp - 1.0) * RU / W)
        dU = np.sum(u * fy) + cv * fT                                # constant volume, adiabatic
        assert abs(dU) <= 1e-10 * (np.sum(np.abs(u * fy)) + 1e-300)


@pytest.mark.parametrize("name", list(MECHS))
def test_mech_integration_conserves_and_reaches_equilibrium(oracle, name):
    m = oracle.Model.mechanism(name)
    table = m.mech.table
    y0, rho = initial_state(m, name)
    W = m.mech.W
    cp0, h0, _ = nasa(table, y0[-1])
    U0 = np.sum((h0 - 1.0) * RU * y0[-1] / W * y0[:-1])
    y, st, _ = oracle.integrate(m, y0, 0.0, 0.2, 1e-10, 1e-20, rho, mxstep=100000)
    assert st["status"] == 0
    assert abs(y[:-1].sum() - 1.0) <= 1e-13
    cp, h, s = nasa(table, y[-1])
    U = np.sum((h - 1.0) * RU * y[-1] / W * y[:-1])
    assert abs(U - U0) <= 1e-6 * np.sum(np.abs((h - 1.0) * RU * y[-1] / W * y[:-1]))
    # detailed balance: sum_k nu_k mu_k / RT = 0, mu/RT = g/RT + ln(C R T / patm)
    T = y[-1]
    C = rho * y[:-1] / W
    sp = [x["name"] for x in table["species"]]
    mu = (h - s) + np.log(np.maximum(C, 1e-300) * RU * T / PATM)
    checked = 0
    for rx in table["reactions"]:
        names = rx["reactants"] + rx["products"]
        if min(C[sp.index(k)] for k in names) < 1e-14:
            continue
        dmu = sum(mu[sp.index(k)] for k in rx["products"]) - sum(mu[sp.index(k)] for k in rx["reactants"])
        assert abs(dmu) < 1e-3, rx["equation"]
        checked += 1
    assert checked >= 8


def kwh_rates(T):
    """KWH96 Table 2 rates as restated in SURVEY.md Appendix B."""
    sT = math.sqrt(T)
    T3, T5, T6 = T / 1e3, T / 1e5, T / 1e6
    S5 = 1.0 / (1.0 + math.sqrt(T5))
    return dict(
        aHp=8.40e-11 / sT * T3**-0.2 / (1 + T6**0.7),
        aHep=1.50e-10 * T**-0.6353,
        ad=1.9e-3 * T**-1.5 * math.exp(-470000 / T) * (1 + 0.3 * math.exp(-94000 / T)),
        aHepp=3.36e-10 / sT * T3**-0.2 / (1 + T6**0.7),
        GH0=5.85e-11 * sT * math.exp(-157809.1 / T) * S5,
        GHe0=2.38e-11 * sT * math.exp(-285335.4 / T) * S5,
        GHep=5.68e-12 * sT * math.exp(-631515.0 / T) * S5)


@pytest.mark.parametrize("photo", [False, True])
@pytest.mark.parametrize("logT", [4.0, 4.5, 5.0, 5.5, 6.5])
def test_kwh_ionisation_equilibrium(oracle, photo, logT):
    kw = {} if photo else dict(gph=(0.0, 0.0, 0.0), eph=(0.0, 0.0, 0.0))
    m = oracle.Model.nyx_kwh(**kw)
    mp, kB = 1.67262192369e-24, 1.380649e-16
    rho = 2.69e-29 * 50
    e = 10**logT * kB / ((5 / 3 - 1) * 0.6 * mp)
    st, r = oracle.kwh_state(m, e, rho)
    assert r == 0
    p = m.kwh
    R = kwh_rates(st["T"])
    nH = p["X"] * rho / mp
    yHe = p["Y"] / (4 * p["X"])
    ne = st["ne"]
    gph = p["gph"]
    # eqs 33-38 at the converged n_e
    assert st["nH0"] / nH == pytest.approx(R["aHp"] / (R["aHp"] + R["GH0"] + gph[0] / ne), rel=1e-10)
    assert st["nHep"] / st["nHe0"] == pytest.approx((R["GHe0"] + gph[1] / ne) / (R["aHep"] + R["ad"]), rel=1e-10)
    assert st["nHepp"] / st["nHep"] == pytest.approx((R["GHep"] + gph[2] / ne) / R["aHepp"], rel=1e-10)
    assert st["nHe0"] + st["nHep"] + st["nHepp"] == pytest.approx(yHe * nH, rel=1e-12)
    # charge neutrality at the root, within the stopping tolerance
    assert (st["nHp"] + st["nHep"] + 2 * st["nHepp"]) / nH == pytest.approx(ne / nH, abs=1e-10)
    # mu and T consistent with x_e
    xe = ne / nH
    mu = (1 + 4 * yHe) / (1 + yHe + xe)
    assert st["T"] == pytest.approx((5 / 3 - 1) * mu * mp * e / kB, rel=1e-14)


def test_kwh_pure_function_and_failure(oracle):
    m = oracle.Model.nyx_kwh()
    f1, _ = oracle.rhs(m, [2e12], 1e-27)
    f2, _ = oracle.rhs(m, [2e12], 1e-27)
    assert f1[0] == f2[0]
    assert oracle.rhs(m, [0.0], 1e-27)[1] == 1
    assert oracle.rhs(m, [1e30], 1e-27)[1] == 1


# ---- difference-quotient Jacobian (CVODE cvLsDenseDQJac) -------------------
def test_jac_dq_exact_on_linear_and_close_on_robertson(oracle):
    """DQ columns of a linear f are the exact matrix up to the rounding of one difference quotient; on
    Robertson (polynomial f) the DQ Jacobian agrees with the analytic one to O(sqrt(u)) relative."""
    lam = [-1.0, -10.0, -1e4]
    m = oracle.Model.linear(lam)
    y = np.array([1.0, 0.5, 2.0])
    fy, _ = oracle.rhs(m, y)
    J, r = oracle.jac_dq(m, y, fy, 1.0 / (1e-6 * np.abs(y) + 1e-10), 1e-3)
    assert r == 0
    assert np.allclose(J, np.diag(lam), rtol=1e-6, atol=0.0)
    rob = oracle.Model.robertson()
    for y in ([0.9, 2e-5, 0.1], [0.3, 1e-6, 0.7], [0.999, 3e-5, 1e-3]):   # interior states (all y_i > 0)
        y = np.array(y)
        fy, _ = oracle.rhs(rob, y)
        Jd, r = oracle.jac_dq(rob, y, fy, 1.0 / (1e-6 * np.abs(y) + 1e-10), 1e-4)
        Ja, _ = oracle.jac(rob, y)
        # row-scaled, with a floor for all-zero rows: a zero analytic entry (e.g. d(y3')/dy2 = 6e7 y2 at
        # y2 = 0) is matched only up to the O(inc) truncation term f'' inc of the one-sided quotient
        scale = np.maximum(np.abs(Ja).max(axis=1, keepdims=True), 1e-3 * np.abs(Ja).max())
        assert r == 0 and np.all(np.abs(Jd - Ja) <= 1e-6 * scale)


@pytest.mark.parametrize("mech", ["h2_lidryer", "drm19_class"])
def test_dq_integration_matches_analytic_ac8(oracle, mech):
    """SPEC AC8: end states with the difference-quotient Jacobian (approaches 3A/3B) agree with the
    analytic-Jacobian run (2A/2B) within 100 rtol on flame cells (modified Newton tolerates J errors; the
    error test guards the accuracy)."""
    from synth import flame_field
    y, rho, F, prog = flame_field(mech, 8, dt=1e-5)
    idx = np.arange(0, y.shape[1], 8)
    m = oracle.Model.mechanism(mech)
    ya, sa = oracle.integrate_batch(m, y, 0.0, 1e-5, 1e-6, 1e-10, rho=rho, fext_yc=F, cells=idx, threads=8)
    yd, sd = oracle.integrate_batch(m, y, 0.0, 1e-5, 1e-6, 1e-10, rho=rho, fext_yc=F, cells=idx, threads=8,
                                    ls=oracle.LS_DENSE_DQ)
    assert np.all(sa["status"] == 0) and np.all(sd["status"] == 0)
    assert np.all(np.abs(yd - ya) <= 100 * 1e-6 * np.abs(ya) + 1e-9)
