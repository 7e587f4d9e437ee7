"""Pins for the oracle primitives (WRMS Eq. 3, dense LU, BDF coefficients).

Each check compares the oracle with something other than itself: SPEC worked
examples (tests/golden/spec_examples.json), exact summation (math.fsum),
brute-force Gaussian elimination written here independently, numpy.linalg,
and the textbook fixed-step BDF coefficients (Byrne & Hindmarsh 1975;
Hairer & Wanner II, III.1)."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def test_wrms_spec_examples(oracle):
    g = json.load(open(GOLD))
    for ex in g["wrms"]:
        assert oracle.wrms(ex["v"], ex["w"]) == pytest.approx(ex["norm"], rel=1e-15, abs=0)


@pytest.mark.parametrize("group", [1, 2, 4, 8, 16, 32])
def test_wrms_any_summation_order_is_exact_to_rounding(oracle, group):
    rng = np.random.default_rng(group)
    for n in (1, 3, 10, 22, 31):
        v = rng.standard_normal(n) * 10.0 ** rng.uniform(-5, 5, n)
        w = 10.0 ** rng.uniform(-3, 3, n)
        exact = math.sqrt(math.fsum((float(a) * float(b)) ** 2 for a, b in zip(v, w)) / n)
        assert oracle.wrms(v, w, group) == pytest.approx(exact, rel=4 * n * 2.0**-52)
        # symmetry: w_i v_i = 1 for all i -> 1
        assert oracle.wrms(1.0 / w, w, group) == pytest.approx(1.0, rel=1e-15)
        # homogeneity ||c v|| = |c| ||v|| (power-of-two c keeps it exact)
        assert oracle.wrms(-8.0 * v, w, group) == 8.0 * oracle.wrms(v, w, group)


def fma(a, b, c):
    """Exactly rounded fused multiply-add via rational arithmetic."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def brute_lu(M):
    """Independent Gaussian elimination with row pivoting (first max), numpy only."""
    A = np.array(M, dtype=np.float64)
    n = len(A)
    piv = []
    for k in range(n):
        p = k + int(np.argmax(np.abs(A[k:, k])))
        piv.append(p)
        A[[k, p]] = A[[p, k]]
        for i in range(k + 1, n):
            A[i, k] = A[i, k] * (1.0 / A[k, k])
            for j in range(k + 1, n):
                A[i, j] = fma(-A[i, k], A[k, j], A[i, j])
    return A, np.array(piv, dtype=np.int32)


def test_lu_spec_examples(oracle):
    g = json.load(open(GOLD))
    for ex in g["lu"]:
        LU, piv, info = oracle.lu_factor(ex["M"])
        assert info == 0
        x = oracle.lu_solve(LU, piv, ex["b"])
        np.testing.assert_allclose(x, ex["x"], rtol=0, atol=1e-15)
        if "piv" in ex:
            assert list(piv) == ex["piv"]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_lu_matches_brute_force_pivots_and_values(oracle, n):
    rng = np.random.default_rng(100 + n)
    for trial in range(50):
        M = rng.standard_normal((n, n)) * 10.0 ** rng.uniform(-3, 3, (n, 1))
        LU, piv, info = oracle.lu_factor(M)
        assert info == 0
        LUb, pivb = brute_lu(M)
        assert np.array_equal(piv, pivb)
        assert np.array_equal(LU, LUb)          # same op order -> bit identical
        b = rng.standard_normal(n)
        x = oracle.lu_solve(LU, piv, b)
        np.testing.assert_allclose(x, np.linalg.solve(M, b), rtol=1e-9 * np.linalg.cond(M))
        # backward error <= c n u
        r = M @ x - b
        assert np.linalg.norm(r, np.inf) <= 8 * n * 2.0**-52 * np.linalg.norm(M, np.inf) * np.linalg.norm(x, np.inf) + 1e-300


def test_lu_singular_is_reported(oracle):
    M = np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 6.0], [0.0, 0.0, 0.0]])
    _, _, info = oracle.lu_factor(M)
    assert info > 0
    _, _, info = oracle.lu_factor(np.zeros((2, 2)))
    assert info == 1


# textbook fixed-step BDF in Nordsieck form (Byrne-Hindmarsh): l / l[0]
L_TEXTBOOK = {
    1: [1, 1],
    2: [1, Fraction(3, 2), Fraction(1, 2)],
    3: [1, Fraction(11, 6), 1, Fraction(1, 6)],
    4: [1, Fraction(25, 12), Fraction(35, 24), Fraction(5, 12), Fraction(1, 24)],
    5: [1, Fraction(137, 60), Fraction(15, 8), Fraction(17, 24), Fraction(1, 8), Fraction(1, 120)],
}
BETA0 = {1: 1, 2: Fraction(2, 3), 3: Fraction(6, 11), 4: Fraction(12, 25), 5: Fraction(60, 137)}
# |error constant| of BDF-q, C_{q+1} = 1/(q+1) * beta0 (Hairer-Wanner III.1, Table 1.1 scaled)
ERRC = {1: Fraction(1, 2), 2: Fraction(2, 9), 3: Fraction(3, 22), 4: Fraction(12, 125), 5: Fraction(10, 137)}


@pytest.mark.parametrize("q", [1, 2, 3, 4, 5])
def test_bdf_coefficients_constant_step(oracle, q):
    h = 0.37
    l, tq = oracle.set_bdf(q, h, [h] * 6, qwait=1)
    np.testing.assert_allclose(l[: q + 1] / l[0], [float(c) for c in L_TEXTBOOK[q]], rtol=1e-14)
    assert 1.0 / l[1] == pytest.approx(float(BETA0[q]), rel=1e-14)          # gamma/h = beta0
    assert tq[2] == pytest.approx(float(ERRC[q]), rel=1e-13)                # LTE constant
    assert tq[5] == pytest.approx(math.factorial(q + 1), rel=1e-13)
    assert tq[4] == pytest.approx(0.1 / tq[2], rel=1e-15)                   # Eq. 4: c_eps * eps


@pytest.mark.parametrize("q", [2, 3, 4, 5])
def test_bdf_coefficients_variable_step_flc_polynomial(oracle, q):
    """Fixed-leading-coefficient BDF (Jackson & Sacks-Davis 1980; the CVODE form):
    l(x) = sum l_i x^i = (1 + x/xi*) prod_{i=1}^{q-1} (1 + x/xi_i), xi_i = (t_n - t_{n-i})/h,
    1/xi* = sum_{j=1}^{q} 1/j - sum_{i=1}^{q-1} 1/xi_i  (so that l_1 = sum 1/j).
    Built here by numpy polynomial products (independent of the recurrences)."""
    rng = np.random.default_rng(q)
    h = 0.1
    tau = list(h * rng.uniform(0.3, 3.0, 6))
    l, _ = oracle.set_bdf(q, h, tau, qwait=2)
    xis = [(h + sum(tau[: i - 1])) / h for i in range(1, q)]
    inv_star = sum(1.0 / j for j in range(1, q + 1)) - sum(1.0 / x for x in xis)
    poly = np.array([1.0])
    for x in xis:
        poly = np.polymul(poly, [1.0 / x, 1.0])
    poly = np.polymul(poly, [inv_star, 1.0])
    np.testing.assert_allclose(l[: q + 1], poly[::-1], rtol=1e-13)
    assert l[1] == pytest.approx(sum(1.0 / j for j in range(1, q + 1)), rel=1e-14)


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 6, 7])
def test_root_matches_high_precision_root(oracle, L):
    """Reading R25: x^(1/L) by a fixed IEEE sequence, within 12 ulp of the exact real root."""
    from decimal import Decimal, getcontext
    getcontext().prec = 60
    rng = np.random.default_rng(L)
    for x in np.concatenate([10.0 ** rng.uniform(-300, 300, 300), rng.uniform(1e-8, 1e4, 300)]):
        exact = float(Decimal(float(x)) ** (Decimal(1) / Decimal(L)))
        assert abs(oracle.root(x, L) - exact) <= 12 * np.spacing(exact)
    for a in (0.5, 2.0, 3.0, 1.25, 7.0):
        assert oracle.root(a ** L, L) == pytest.approx(a, rel=2e-16)
    assert oracle.root(0.0, L) == 0.0


# ---- typical-value tolerances (Eq. 7) -----------------
def test_typical_values_spec_examples(oracle):
    g = json.load(open(GOLD))
    for ex in g["typical_values"]:
        y = np.array([ex["component"]])
        assert oracle.typical_values(y)[0] == ex["tv"], ex["tag"]
    for ex in g["atol_from_typical"]:
        a = oracle.atol_from_typical([ex["tv"]], ex["eta"], ex["floor"])[0]
        assert a == pytest.approx(ex["atol"], rel=1e-15, abs=0.0), ex["tag"]


def test_typical_values_brute_force_and_invariances(oracle):
    """Midpoint of the range by an independent numpy scan; invariant under permutation of the cells and under
    duplication of a cell inside [min, max]; an exact midpoint when min and max are dyadic."""
    rng = np.random.default_rng(5)
    y = rng.standard_normal((7, 513)) * 10.0 ** rng.uniform(-12, 3, (7, 1))
    tv = oracle.typical_values(y)
    ref = 0.5 * (y.min(axis=1) + y.max(axis=1))
    assert np.array_equal(tv, ref)
    perm = rng.permutation(y.shape[1])
    assert np.array_equal(oracle.typical_values(y[:, perm]), tv)
    dup = np.concatenate([y, y[:, [3, 3, 100]]], axis=1)
    assert np.array_equal(oracle.typical_values(dup), tv)
    z = np.array([[0.25, -1.5, 4.0, 0.5]])
    assert oracle.typical_values(z)[0] == 1.25            # (-1.5 + 4) / 2, exact


def test_atol_from_typical_properties(oracle):
    """Eq. 7 scaling: atol proportional to tv above the floor; tv defaults to 1 -> atol = eta."""
    tv = np.array([1.0, 2500.0, 0.0, 1e-40, 3.0])
    a = oracle.atol_from_typical(tv, 1e-6, 1e-30)
    assert a[0] == 1e-6 and a[2] == 1e-30 and a[3] == 1e-30
    assert a[4] == 1e-6 * 3.0
    assert np.array_equal(oracle.atol_from_typical(np.ones(4), 1e-10, 1e-30), np.full(4, 1e-10))
