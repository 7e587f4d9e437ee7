"""Pins for the oracle integrator: closed form of
y' = lambda y, exact scale invariance, published Robertson values
(tests/golden/robertson_reference.json) plus an independent scipy Radau
solution, linear-invariant conservation, the Nordsieck interpolation
invariant, Newton behaviour on linear problems, tolerance monotonicity and
failure statuses."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "robertson_reference.json")


@pytest.mark.parametrize("rtol", [1e-4, 1e-6, 1e-8])
def test_linear_decay_closed_form(oracle, rtol):
    m = oracle.Model.linear([-1.0])
    y, st, _ = oracle.integrate(m, [1.0], 0.0, 1.0, rtol, 1e-12)
    exact = np.exp(-1.0)
    assert st["status"] == 0 and st["t_reached"] == 1.0
    assert abs(y[0] - exact) <= 10 * (rtol * exact + 1e-12)


def test_linear_system_closed_form_multi_component(oracle):
    lam = np.array([-1.0, -10.0, -1e3, 0.5])
    m = oracle.Model.linear(lam)
    y0 = np.array([1.0, 2.0, -3.0, 0.25])
    y, st, _ = oracle.integrate(m, y0, 0.0, 2.0, 1e-7, 1e-12)
    exact = y0 * np.exp(lam * 2.0)
    assert np.all(np.abs(y - exact) <= 10 * (1e-7 * np.abs(exact) + 1e-12))


def test_scale_invariance(oracle):
    """(lambda, tf) -> (c lambda, tf/c) with c a power of two is an exact symmetry of the
    algorithm: every h scales by c^-1 exactly, so y and all counters are identical."""
    a, sa, _ = oracle.integrate(oracle.Model.linear([-1.0]), [1.0], 0.0, 1.0, 1e-6, 1e-12)
    b, sb, _ = oracle.integrate(oracle.Model.linear([-1024.0]), [1.0], 0.0, 1.0 / 1024, 1e-6, 1e-12)
    assert a[0] == b[0]
    for k in ("nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn", "q_last"):
        assert sa[k] == sb[k], k
    assert sa["h_last"] == sb["h_last"] * 1024


def test_linear_newton_converges_in_at_most_two_iterations(oracle):
    m = oracle.Model.linear([-3.0, -300.0, -3e4])
    y, st, _ = oracle.integrate(m, [1.0, 1.0, 1.0], 0.0, 1.0, 1e-6, 1e-12)
    attempts = st["nst"] + st["netf"] + st["ncfn"]
    assert st["ncfn"] == 0
    assert st["nni"] <= 2 * attempts


@pytest.mark.parametrize("t", ["0.4", "4", "40"])
@pytest.mark.parametrize("tol", [(1e-6, 1e-10), (1e-4, (1e-8, 1e-14, 1e-6))])
def test_robertson_published_values(oracle, t, tol):
    g = json.load(open(GOLD))
    ref = np.array(g["values"][t])
    rtol, atol = tol
    y, st, _ = oracle.integrate(oracle.Model.robertson(), g["y0"], 0.0, float(t), rtol, atol)
    assert st["status"] == 0
    err = np.abs(y - ref) / (rtol * np.abs(ref) + np.asarray(atol))
    assert err.max() <= 5.0, err
    # conservation of y1+y2+y3 (c.f = 0 => exact to rounding, §8c.4)
    assert abs(y.sum() - 1.0) <= 4e-15


def test_robertson_against_independent_radau(oracle):
    scipy_integrate = pytest.importorskip("scipy.integrate")
    k1, k2, k3 = 0.04, 3e7, 1e4

    def f(t, y):
        return [-k1 * y[0] + k3 * y[1] * y[2], k1 * y[0] - k3 * y[1] * y[2] - k2 * y[1] ** 2, k2 * y[1] ** 2]

    def jac(t, y):
        return [[-k1, k3 * y[2], k3 * y[1]], [k1, -k3 * y[2] - 2 * k2 * y[1], -k3 * y[1]], [0, 2 * k2 * y[1], 0]]

    y0 = [0.97, 2e-5, 0.03 - 2e-5]
    sol = scipy_integrate.solve_ivp(f, (0, 40), y0, method="Radau", rtol=1e-12, atol=1e-16, jac=jac)
    ref = sol.y[:, -1]
    y, st, _ = oracle.integrate(oracle.Model.robertson(), y0, 0.0, 40.0, 1e-6, 1e-10)
    assert np.all(np.abs(y - ref) <= 10 * (1e-6 * np.abs(ref) + 1e-10))
    # the oracle's analytic J is the derivative of its RHS (central differences)
    yy = np.array([0.7, 3e-5, 0.29])
    J, _ = oracle.jac(oracle.Model.robertson(), yy)
    for j in range(3):
        h = 1e-6 * max(abs(yy[j]), 1e-6)
        e = np.zeros(3)
        e[j] = h
        fd = (oracle.rhs(oracle.Model.robertson(), yy + e)[0] - oracle.rhs(oracle.Model.robertson(), yy - e)[0]) / (2 * h)
        np.testing.assert_allclose(J[:, j], fd, rtol=1e-6, atol=1e-6 * np.abs(J).max())


def test_robertson_rhs_spec_examples(oracle):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
    for ex in g["robertson_rhs"]:
        f, r = oracle.rhs(oracle.Model.robertson(), ex["y"])
        assert r == 0
        np.testing.assert_allclose(f, ex["f"], rtol=1e-15, atol=0)


def test_nordsieck_interpolation_invariant(oracle):
    """After every accepted step P(t) = sum_j zn[j] ((t - t_n)/h)^j reproduces the last q
    accepted solutions y_n..y_{n-q+1} (FLC Nordsieck invariant, §8c.4)."""
    m = oracle.Model.robertson()
    y, st, tr = oracle.integrate(m, [1.0, 0.0, 0.0], 0.0, 40.0, 1e-6, 1e-10, trace=2000)
    assert len(tr["tn"]) == st["nst"]
    ys = tr["zn"][:, 0, :]
    worst = 0.0
    for k in range(10, len(tr["tn"])):
        q, h, tn = tr["q"][k], tr["h"][k], tr["tn"][k]
        for j in range(1, q):
            s = (tr["tn"][k - j] - tn) / h
            P = sum(tr["zn"][k, i, :] * s**i for i in range(q + 1))
            tol = 1e-6 * np.abs(ys[k - j]) + 1e-10
            worst = max(worst, float(np.max(np.abs(P - ys[k - j]) / tol)))
    assert worst < 1e-6, worst


def test_tolerance_monotonicity(oracle):
    m = oracle.Model.linear([-1.0])
    errs = []
    for rtol in (1e-3, 1e-5, 1e-7, 1e-9):
        y, _, _ = oracle.integrate(m, [1.0], 0.0, 1.0, rtol, 1e-14)
        errs.append(abs(y[0] - np.exp(-1)))
    assert all(b < a for a, b in zip(errs, errs[1:]))


def test_failure_statuses(oracle):
    m = oracle.Model.robertson()
    # too much work: mxstep = 5
    y, st, _ = oracle.integrate(m, [1.0, 0.0, 0.0], 0.0, 40.0, 1e-6, 1e-10, mxstep=5)
    assert st["status"] == 1 and st["nst"] == 5 and st["t_reached"] < 40.0
    # non-finite input
    y, st, _ = oracle.integrate(m, [np.nan, 0.0, 0.0], 0.0, 1.0, 1e-6, 1e-10)
    assert st["status"] == 5
    # unresolvable RHS failure from the start (KWH with e <= 0)
    y, st, _ = oracle.integrate(oracle.Model.nyx_kwh(), [-1.0], 0.0, 1e13, 1e-6, 1e-10, rho=1e-28)
    assert st["status"] == 4


def test_batch_driver_matches_single_cell(oracle):
    m = oracle.Model.robertson()
    rng = np.random.default_rng(0)
    N = 64
    a = 3e-5 * rng.random(N)
    b = 0.5 * rng.random(N)
    Y = np.stack([1 - a - b, a, b])
    yb, st = oracle.integrate_batch(m, Y, 0.0, 40.0, 1e-6, 1e-10, threads=4)
    for c in (0, 17, 63):
        y1, s1, _ = oracle.integrate(m, Y[:, c], 0.0, 40.0, 1e-6, 1e-10)
        assert np.array_equal(y1, yb[:, c]) and s1["nst"] == st["nst"][c]


# ---------------------------------------------------------------- global-norm mode
def test_global_mode_identical_cells_reproduce_single_cell(oracle):
    """SPEC AC7: k identical cells integrated as one lockstep batch reproduce the
    single-cell run with the identical step count (batch WRMS of identical blocks = cell WRMS)."""
    m = oracle.Model.robertson()
    y1, s1, _ = oracle.integrate(m, [1.0, 0.0, 0.0], 0.0, 40.0, 1e-6, 1e-10)
    for k in (1, 64, 300):
        Y = np.tile(np.array([[1.0], [0.0], [0.0]]), (1, k))
        yg, sg = oracle.integrate_global(m, Y, 0.0, 40.0, 1e-6, 1e-10)
        assert sg["status"] == 0
        assert sg["nst"] == s1["nst"] and sg["netf"] == s1["netf"] and sg["nje"] == s1["nje"], (k, sg, s1)
        # the only difference is the rounding of the batch sum (k partial sums): ~1e-12 relative
        np.testing.assert_allclose(yg, np.tile(y1[:, None], (1, k)), rtol=1e-11, atol=1e-300)


def test_global_mode_linear_closed_form(oracle):
    lam = np.array([-1.0, -5.0, -25.0, -125.0])
    m = oracle.Model.linear([-1.0])
    # a batch of 4 one-component cells with different rates is not expressible with one
    # model, so use a 4-component linear cell and a batch of 3 copies with different y0
    m = oracle.Model.linear(lam)
    Y = np.stack([np.linspace(1.0, 2.0, 3)] * 4)
    yg, sg = oracle.integrate_global(m, Y, 0.0, 1.0, 1e-7, 1e-12)
    exact = Y * np.exp(lam[:, None])
    assert sg["status"] == 0
    assert np.all(np.abs(yg - exact) <= 20 * (1e-7 * np.abs(exact) + 1e-12))


def test_global_mode_lockstep_costs_more_than_per_cell(oracle):
    """in lockstep the effort is dictated by the most difficult cells: the batch takes at
    least as many steps as its hardest cell, and each step advances every cell."""
    from synth import robertson_field
    Y = robertson_field(32)
    _, st = oracle.integrate_batch(oracle.Model.robertson(), Y, 0.0, 40.0, 1e-6, 1e-10)
    yg, sg = oracle.integrate_global(oracle.Model.robertson(), Y, 0.0, 40.0, 1e-6, 1e-10)
    assert sg["status"] == 0
    assert sg["nst"] >= 0.5 * st["nst"].max()
    assert np.abs(yg.sum(axis=0) - 1.0).max() <= 1e-14       # conservation per cell
