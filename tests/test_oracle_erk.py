"""Pins for the oracle's explicit adaptive ERK (oracle/erk.c, reading R30).

Nothing here restates the tableau: one step on y' = lambda y must equal the degree-4 Taylor polynomial of
e^{h lambda} (the stability function of any 4-stage order-4 method, here the classical RK4 weights); the
global error at fixed h must fall at rate 4 (SPEC AC2); the embedded estimate must be O(h^4); an
adaptive run must meet the tolerance against the closed form; on an ignition cell the explicit method must
take many more steps than BDF (the direction of P:426, SPEC AC4 S:598)."""
import numpy as np
import pytest


@pytest.mark.parametrize("z", [-0.5, -0.1, 0.01, 0.3, -2.0, -2.7])
def test_one_step_is_taylor_degree_four(oracle, z):
    m = oracle.Model.linear([z])
    yn, err, st, nfe = oracle.erk_step(m, [1.0], 1.0)
    R = 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24
    assert st == 0 and nfe == 5
    assert abs(yn[0] - R) <= 4 * np.finfo(float).eps * max(1.0, abs(R))
    # the estimate is the difference to a third-order solution: it vanishes to O(z^4) and not to O(z^5)
    assert abs(err[0]) <= 1.0 * abs(z) ** 4 and abs(err[0]) >= 1e-3 * abs(z) ** 4


def test_global_order_four_at_fixed_step(oracle):
    """y' = -y on [0, 1] with a fixed step: error ratio 2^4 on halving h, rate 4 +- 0.25."""
    m = oracle.Model.linear([-1.0])
    errs = []
    for nsteps in (10, 20, 40):
        y = np.array([1.0])
        for _ in range(nsteps):
            y, _, st, _ = oracle.erk_step(m, y, 1.0 / nsteps)
        errs.append(abs(y[0] - np.exp(-1.0)))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(rates - 4.0) <= 0.25), rates


def test_error_estimate_is_fourth_order_in_h(oracle):
    """The embedded (order-3) difference is O(h^4): halving h divides it by ~16, on a linear and on a
    nonlinear (Robertson, non-stiff start) right-hand side."""
    m = oracle.Model.linear([-1.0, 2.0])
    e1 = oracle.erk_step(m, [1.0, 1.0], 0.02)[1]
    e2 = oracle.erk_step(m, [1.0, 1.0], 0.01)[1]
    assert np.all(np.abs(np.log2(np.abs(e1 / e2)) - 4.0) < 0.1)
    r = oracle.Model.robertson()
    y0 = np.array([0.9, 0.0, 0.1])
    e1 = oracle.erk_step(r, y0, 2e-6)[1]
    e2 = oracle.erk_step(r, y0, 1e-6)[1]
    k = np.abs(e1) > 1e-30
    assert np.all(np.abs(np.log2(np.abs(e1[k] / e2[k])) - 4.0) < 0.2)


@pytest.mark.parametrize("rtol", [1e-4, 1e-6, 1e-8])
def test_adaptive_closed_form(oracle, rtol):
    lam = np.array([-1.0, -5.0, 0.5, -20.0])
    m = oracle.Model.linear(lam)
    y0 = np.array([1.0, -2.0, 0.5, 3.0])
    y, st, _ = oracle.integrate(m, y0, 0.0, 2.0, rtol, 1e-12, method=oracle.METHOD_ERK4)
    exact = y0 * np.exp(2.0 * lam)
    assert st["status"] == 0 and st["t_reached"] == 2.0 and st["q_last"] == 4
    assert np.all(np.abs(y - exact) <= 10 * (rtol * np.abs(exact) + 1e-12))
    assert st["nje"] == 0 and st["nni"] == 0 and st["nsetups"] == 0     # no algebraic solver
    attempts = st["nst"] + st["netf"]
    assert 4 * attempts + 2 <= st["nfe"] <= 5 * attempts + 2 + st["nst"]


def test_tolerance_monotonicity(oracle):
    m = oracle.Model.linear([-3.0])
    errs = []
    for rtol in (1e-4, 1e-6, 1e-8):
        y, st, _ = oracle.integrate(m, [1.0], 0.0, 1.0, rtol, 1e-14, method=oracle.METHOD_ERK4)
        errs.append(abs(y[0] - np.exp(-3.0)))
    assert errs[1] < errs[0] and errs[2] < errs[1]


def test_zero_rhs_keeps_state(oracle):
    m = oracle.Model.linear([0.0, 0.0])
    y, st, _ = oracle.integrate(m, [1.0, -2.0], 0.0, 5.0, 1e-6, 1e-10, method=oracle.METHOD_ERK4)
    assert st["status"] == 0 and np.array_equal(y, [1.0, -2.0]) and st["netf"] == 0


def test_stiff_explicit_needs_many_more_steps(oracle):
    """P:426 direction (SPEC AC4): on reacting and burnt flame cells over one CFD step (dt 1e-5 s) the explicit method takes
    >= 10x the steps of BDF; its RHS evaluations per step stay near the 5 stages."""
    import synth
    yf, rho, F, prog = synth.flame_field("h2_lidryer", 16, cells=np.arange(4096))
    react = np.concatenate([np.where((prog > 0.1) & (prog < 0.9))[0][:2], np.where(prog > 0.98)[0][:2]])
    assert len(react) == 4
    m = oracle.Model.mechanism("h2_lidryer")
    kw = dict(rho=rho[react], fext_yc=F[:, react])
    ye, se = oracle.integrate_batch(m, yf[:, react], 0.0, 1e-5, 1e-6, 1e-10, method=oracle.METHOD_ERK4,
                                    mxstep=100000, **kw)
    yb, sb = oracle.integrate_batch(m, yf[:, react], 0.0, 1e-5, 1e-6, 1e-10, **kw)
    assert np.all(se["status"] == 0) and np.all(sb["status"] == 0)
    assert se["nst"].sum() >= 10 * sb["nst"].sum()
    rhs_per_step = se["nfe"].sum() / se["nst"].sum()
    assert 5.0 <= rhs_per_step <= 6.5
    assert np.all(np.abs(ye - yb) <= 100 * (1e-6 * np.abs(yb) + 1e-10))
