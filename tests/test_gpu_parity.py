"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on identical
seeded inputs.

Bars (written in each test): LU factor/solve bit-identical (integer pivots
equal); RHS |f_gpu - f_orc| <= 1e-12 S_i (reading R19); Jacobian row-scaled
<= 1e-12 vs the oracle's complex-step J; integrated end states
|dy| <= 10 (rtol |y| + atol) per cell and component plus the conservation
check on both sides."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2405_01713_b200 as P  # noqa: E402
from synth import flame_field, nyx_field, robertson_field, uniform  # noqa: E402
from synth.fields import stratified_sample  # noqa: E402

DEV = torch.device("cuda", 0)
STAT_KEYS = ("nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn")
MECH = {"h2": ("h2_lidryer", 10), "drm19": ("drm19_class", 22), "gri53": ("gri53_class", 54)}
KERNELS = ("split", "thread", "group")   # per-cell kernel organisations of the mechanism models (bdfb_set_kernel)


def cu(a):
    return None if a is None else torch.tensor(np.ascontiguousarray(a), device=DEV)


def end_state_check(yg, yo, rtol, atol, frac_min=0.0):
    tol = 10.0 * (rtol * np.abs(yo) + atol)
    err = np.abs(yg - yo)
    ok = err <= tol
    assert ok.all(), f"{(~ok.all(axis=0)).sum()} cells outside 10 tol; worst {np.max(err / tol):.3g}"


def run_gpu(model, n, y0, t1, rtol, atol, rho=None, F=None, layout="YC", kernel="auto", **kw):
    """Integrate on the GPU; st carries the aggregate stats plus "group", the WRMS lane-group
    size (reading R15) of the kernel used, which the oracle reproduces."""
    N = y0.shape[1]
    b = P.Batch(N, n, rtol, atol, **kw)
    b.set_kernel(kernel)
    b.set_model(model)
    cs = b.attach_cell_stats()
    y = cu(y0 if layout == "YC" else y0.T)
    b.integrate(0.0, t1, y, f_ext=cu(F if (F is None or layout == "YC") else F.T), aux=cu(rho), layout=layout)
    st = b.stats()
    st["group"] = b.wrms_group
    yy = y.cpu().numpy()
    return (yy if layout == "YC" else yy.T), {k: v.cpu().numpy() for k, v in cs.items()}, st


# ------------------------------------------------------------------ LU
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 22, 32])
def test_lu_bit_identical(oracle, n):
    rng = np.random.default_rng(n)
    N = 1000 + 37  # several warps + a ragged tail
    M = rng.standard_normal((n, n, N)) * 10.0 ** rng.uniform(-3, 3, (n, 1, N))
    b = rng.standard_normal((n, N))
    if n > 1:
        M[:, :, 5] = M[:, :, 6]
        M[0, :, 5] = M[1, :, 5]              # exact duplicate rows: pivot ties
        M[:, 0, 7] = 0.0                      # singular column
    LU, piv, x, info = (t.cpu().numpy() for t in P.lu_factor_solve(cu(M), cu(b)))
    for c in range(N):
        LUo, pivo, io = oracle.lu_factor(M[:, :, c])
        assert info[c] == io, c
        if io:
            continue
        assert np.array_equal(piv[:, c], pivo), c
        assert np.array_equal(LU[:, :, c], LUo), c
        assert np.array_equal(x[:, c], oracle.lu_solve(LUo, pivo, b[:, c])), c


@pytest.mark.parametrize("n", [2, 4, 8, 10, 16, 22, 32])
def test_split_lu_bit_identical(oracle, n):
    """The default SPLIT integrator's own LU (oct_factor, 8 lanes per cell, K_lu's record layout) and the
    substitutions of its Newton solve (K_ctl) vs LU_FACTOR / LU_SOLVE: identical pivots, bit-identical
    factors and solutions (reading R16), pivot ties and exact zero pivots included (north_star: LU solve
    within 1e-12 on identical inputs; this is exact)."""
    rng = np.random.default_rng(1000 + n)
    N = 4096 + 29
    M = rng.standard_normal((n, n, N)) * 10.0 ** rng.uniform(-3, 3, (n, 1, N))
    b = rng.standard_normal((n, N))
    M[:, :, 5] = M[:, :, 6]
    M[0, :, 5] = M[1, :, 5]                  # exact duplicate rows: pivot ties
    M[:, 0, 7] = 0.0                          # zero first column: singular at k = 0
    M[:, n // 2, 8] = 0.0                     # singular later
    M[:, :, 9] = np.abs(M[:, :, 9])           # all-positive: ties in |.| broken by position only
    M[1, 0, 10] = -M[0, 0, 10]                # |a| tie between rows 0 and 1
    LU, piv, x, info = (t.cpu().numpy() for t in P.lu_factor_solve(cu(M), cu(b), routine="split"))
    for c in range(N):
        LUo, pivo, io = oracle.lu_factor(M[:, :, c])
        assert info[c] == io, c
        if io:
            continue
        assert np.array_equal(piv[:, c], pivo), c
        assert np.array_equal(LU[:, :, c], LUo), c
        assert np.array_equal(x[:, c], oracle.lu_solve(LUo, pivo, b[:, c])), c
        if c % 512 == 0:   # and within rounding of the plain (true-division) solve
            np.testing.assert_allclose(x[:, c], oracle.lu_solve(LUo, pivo, b[:, c], plain=True),
                                       rtol=1e-12 * max(1.0, float(np.linalg.cond(M[:, :, c]))) , atol=0)


# ------------------------------------------------------------------ RHS / J
def model_states(name, count, seed=7):
    if name == "robertson":
        y = robertson_field(count, seed=seed)
        y[1] = 4e-5 * uniform(seed, np.arange(count), 30)
        return y, None, 0.1 * (uniform(seed, np.arange(count), 31) - 0.5)[None, :] * np.ones((3, 1))
    if name == "nyx_kwh":
        L = int(round(count ** (1 / 3)))
        e, rho, fe = nyx_field(L)
        return e, rho, fe
    mech = MECH[name][0]
    L = int(round(count ** (1 / 3)))
    y, rho, F, prog = flame_field(mech, L)
    return y, rho, F


def oracle_model(oracle, name):
    if name == "robertson":
        return oracle.Model.robertson()
    if name == "nyx_kwh":
        return oracle.Model.nyx_kwh()
    return oracle.Model.mechanism(MECH[name][0])


@pytest.mark.parametrize("name,kernel", [("robertson", "thread"), ("nyx_kwh", "thread"), ("h2", "thread"),
                                         ("h2", "group"), ("h2", "split"), ("drm19", "thread"), ("drm19", "group"),
                                         ("drm19", "split"), ("gri53", "auto")])
def test_rhs_parity(oracle, name, kernel):
    y, rho, F = model_states(name, 131072 if name in ("h2", "drm19") and kernel == "split" else 32768)
    n, N = y.shape
    b = P.Batch(N, n, 1e-6, 1e-10)
    b.set_kernel(kernel)
    b.set_model(name)
    f, st = P.eval_rhs(b, cu(y), f_ext=cu(F), aux=cu(rho))
    f, st = f.cpu().numpy(), st.cpu().numpy()
    m = oracle_model(oracle, name)
    # every state for the default kernel of the mechanisms (>= 1e5 states), else a sample
    full = (kernel == "split" and name != "gri53") or N <= 4096
    idx = np.arange(N) if full else np.sort(np.random.default_rng(1).choice(N, 4096, replace=False))
    worst = 0.0
    for c in idx:
        r = rho[c] if rho is not None else 1.0
        fo, ro = oracle.rhs(m, y[:, c], r, None if F is None else F[:, c])
        S, _ = oracle.rhs_scale(m, y[:, c], r, None if F is None else F[:, c])
        assert st[c] == ro
        if ro:
            continue
        d = np.abs(f[:, c] - fo)
        assert np.all(d <= 1e-12 * S + 1e-300), (c, d / (S + 1e-300))
        worst = max(worst, float(np.max(d / (S + 1e-300))))
    print(f"{name}: worst |df|/S = {worst:.3g}")


@pytest.mark.parametrize("name,kernel", [("robertson", "thread"), ("h2", "thread"), ("h2", "group"),
                                         ("h2", "split"), ("drm19", "thread"), ("drm19", "group"),
                                         ("drm19", "split"), ("gri53", "auto")])
def test_jacobian_parity(oracle, name, kernel):
    y, rho, F = model_states(name, 4096)
    n, N = y.shape
    b = P.Batch(N, n, 1e-6, 1e-10)
    b.set_kernel(kernel)
    b.set_model(name)
    J = P.eval_jac(b, cu(y), aux=cu(rho)).cpu().numpy()
    m = oracle_model(oracle, name)
    worst = 0.0
    for c in range(0, N, 7):
        Jo, r = oracle.jac(m, y[:, c], rho[c] if rho is not None else 1.0)
        assert r == 0
        scale = np.abs(Jo).max(axis=1, keepdims=True) + 1e-300
        e = np.abs(J[:, :, c] - Jo) / scale
        assert np.all(e <= 1e-12), (c, np.unravel_index(np.argmax(e), e.shape), e.max())
        worst = max(worst, float(e.max()))
    print(f"{name}: worst row-scaled |dJ| = {worst:.3g}")


# ------------------------------------------------------------------ integration
def test_robertson_c1_bit_identical(oracle):
    """C1 (1024 cells, t in [0, 40], rtol 1e-4): RHS, J, LU, WRMS and step-size root all follow
    the same IEEE operation sequence on both sides, so every cell is bit-identical."""
    y0 = robertson_field(1024)
    for rtol, atol in ((1e-4, (1e-8, 1e-14, 1e-6)), (1e-6, 1e-10)):
        yg, sg, st = run_gpu("robertson", 3, y0, 40.0, rtol, atol)
        yo, so = oracle.integrate_batch(oracle.Model.robertson(), y0, 0.0, 40.0, rtol, atol, threads=8)
        end_state_check(yg, yo, rtol, np.broadcast_to(np.asarray(atol, dtype=float), (3,))[:, None])
        # the plain-arithmetic oracle (libm pow roots, true division): same band, no bit identity expected
        yp, _ = oracle.integrate_batch(oracle.Model.robertson(), y0, 0.0, 40.0, rtol, atol, threads=8, plain=True)
        end_state_check(yg, yp, rtol, np.broadcast_to(np.asarray(atol, dtype=float), (3,))[:, None])
        assert np.abs(yg.sum(axis=0) - y0.sum(axis=0)).max() <= 1e-14
        assert st["n_failed"] == 0 and st["n_cells"] == 1024
        for k in STAT_KEYS:
            assert np.array_equal(sg[k], so[k]), k
        assert np.array_equal(yg, yo)


def test_nyx_c2_parity(oracle):
    e, rho, fe = nyx_field(16)
    dt = 3e15
    yg, sg, st = run_gpu("nyx_kwh", 1, e, dt, 1e-6, 1e-10, rho=rho, F=fe)
    yo, so = oracle.integrate_batch(oracle.Model.nyx_kwh(), e, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=fe, threads=8)
    assert np.array_equal(sg["status"], so["status"])
    ok = sg["status"] == 0
    end_state_check(yg[:, ok], yo[:, ok], 1e-6, 1e-10)
    same = np.mean([all(sg[k][c] == so[k][c] for k in STAT_KEYS) for c in range(e.shape[1])])
    print(f"C2: identical per-cell stats {same:.4f}")


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("name,dt", [("h2", 1e-5), ("h2", 1e-6), ("drm19", 1e-5), ("drm19", 1e-6)])
def test_flame_parity(oracle, name, dt, kernel):
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 16, dt=dt)
    yg, sg, st = run_gpu(name, n, y0, dt, 1e-6, 1e-10, rho=rho, F=F, kernel=kernel)
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F,
                                    group=st["group"], threads=8)
    assert st["n_failed"] == 0
    end_state_check(yg, yo, 1e-6, 1e-10)
    same = np.mean([all(sg[k][c] == so[k][c] for k in STAT_KEYS) for c in range(y0.shape[1])])
    print(f"{name} dt={dt} {kernel}: identical per-cell stats {same:.4f}")
    assert same > 0.95
    if kernel == "split":   # the plain-arithmetic oracle (libm pow roots, true division): same band
        yp, _ = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F,
                                       group=st["group"], threads=8, plain=True)
        end_state_check(yg, yp, 1e-6, 1e-10)


@pytest.mark.parametrize("name", ["h2", "drm19"])
def test_flame_parity_slot_reuse(oracle, name, monkeypatch):
    """SPLIT with a small slot pool (64 slots for 4096 cells): every slot stores a finished cell and loads the
    next one into a dirty record many times; results must equal the oracle's as with one cell per slot."""
    monkeypatch.setenv("BDFB_SPLIT_SLOTS", "64")
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 16, dt=1e-5)
    yg, sg, st = run_gpu(name, n, y0, 1e-5, 1e-6, 1e-10, rho=rho, F=F, kernel="split")
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, 1e-5, 1e-6, 1e-10, rho=rho, fext_yc=F,
                                    group=st["group"], threads=8)
    assert st["n_failed"] == 0 and np.array_equal(sg["status"], so["status"])
    end_state_check(yg, yo, 1e-6, 1e-10)
    monkeypatch.delenv("BDFB_SPLIT_SLOTS")
    yd, _, _ = run_gpu(name, n, y0, 1e-5, 1e-6, 1e-10, rho=rho, F=F, kernel="split")
    assert np.array_equal(yd, yg)         # the pool size never changes a result


def element_matrix(mech):
    """E[j, k] / W_k: moles of element j per gram of species k (problem data: the table's compositions)."""
    t = oracle_table(mech)
    els = sorted({e for s in t["species"] for e in s["composition"]})
    E = np.array([[s["composition"].get(e, 0) / s["W"] for s in t["species"]] for e in els])
    return els, E


def oracle_table(mech):
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "mechanisms",
                                       mech + ".json")))


@pytest.mark.parametrize("name", ["h2", "drm19"])
def test_mass_and_element_conservation_both_sides(oracle, name):
    """F_Y = 0 (only F_T forcing): sum_k Y_k and every element sum sum_k E_jk Y_k / W_k are linear invariants
    (c.f = 0), conserved to round-off on both sides."""
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 8, dt=1e-5)
    yg, _, st = run_gpu(name, n, y0, 1e-5, 1e-6, 1e-10, rho=rho, F=F)
    yo, _ = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, 1e-5, 1e-6, 1e-10, rho=rho,
                                   fext_yc=F, group=st["group"], threads=8)
    s0 = y0[:-1].sum(axis=0)
    assert np.abs(yg[:-1].sum(axis=0) - s0).max() <= 1e-13
    assert np.abs(yo[:-1].sum(axis=0) - s0).max() <= 1e-13
    els, E = element_matrix(mech)
    e0 = E @ y0[:-1]
    scale = np.abs(E) @ np.abs(y0[:-1])
    for side in (yg, yo):
        assert np.all(np.abs(E @ side[:-1] - e0) <= 1e-13 * scale), els


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("kernel", KERNELS)
def test_edge_cases(oracle, kernel):
    y0, rho, F, prog = flame_field("h2_lidryer", 4)        # 64 cells
    y0 = y0[:, :61].copy()                                    # ragged tail
    rho, F = rho[:61].copy(), F[:, :61].copy()
    y0[0, 3] = np.nan                                         # non-finite input
    F[5, 9] = np.inf
    yg, sg, st = run_gpu("h2", 10, y0, 1e-5, 1e-6, 1e-10, rho=rho, F=F, kernel=kernel)
    G = st["group"]
    assert sg["status"][3] == 5 and sg["status"][9] == 5
    assert np.isnan(yg[0, 3]) and np.array_equal(yg[:, 9], y0[:, 9])
    ok = np.ones(61, bool)
    ok[[3, 9]] = False
    yo, so = oracle.integrate_batch(oracle.Model.mechanism("h2_lidryer"), y0, 0.0, 1e-5, 1e-6, 1e-10, rho=rho,
                                    fext_yc=F, group=G)
    assert np.array_equal(so["status"], sg["status"])
    end_state_check(yg[:, ok], yo[:, ok], 1e-6, 1e-10)
    assert st["n_failed"] == 2
    # too much work: mxstep = 3
    yg2, sg2, st2 = run_gpu("h2", 10, y0[:, ok], 1e-5, 1e-6, 1e-10, rho=rho[ok], F=F[:, ok], mxstep=3, kernel=kernel)
    tmw = sg2["status"] == 1
    assert tmw.any() and np.all(sg2["t_reached"][tmw] < 1e-5) and np.all(sg2["nst"][tmw] == 3)
    assert np.all(sg2["status"][~tmw] == 0) and np.all(sg2["nst"][~tmw] <= 3)
    yo2, so2 = oracle.integrate_batch(oracle.Model.mechanism("h2_lidryer"), y0[:, ok], 0.0, 1e-5, 1e-6, 1e-10,
                                      rho=rho[ok], fext_yc=F[:, ok], group=G, mxstep=3)
    assert np.array_equal(so2["status"], sg2["status"])
    end_state_check(yg2, yo2, 1e-6, 1e-10)
    # CY layout == YC layout, bit for bit
    ycy, _, _ = run_gpu("h2", 10, y0[:, ok], 1e-5, 1e-6, 1e-10, rho=rho[ok], F=F[:, ok], layout="CY", kernel=kernel)
    assert np.array_equal(ycy, yg[:, ok])
    # single cell
    y1, s1, _ = run_gpu("robertson", 3, np.array([[1.0], [0.0], [0.0]]), 40.0, 1e-6, 1e-10)
    yo1, _, _ = oracle.integrate(oracle.Model.robertson(), [1.0, 0.0, 0.0], 0.0, 40.0, 1e-6, 1e-10)
    assert np.array_equal(y1[:, 0], yo1)


@pytest.mark.parametrize("kernel", KERNELS)
def test_sharding_invariance_bitwise(kernel):
    """Cells are independent: integrating any subset (what a rank does) gives bit-identical results."""
    y0, rho, F, prog = flame_field("drm19_class", 8, dt=1e-5)
    yall, _, _ = run_gpu("drm19", 22, y0, 1e-5, 1e-6, 1e-10, rho=rho, F=F, kernel=kernel)
    for r in range(3):
        sub = np.arange(r, y0.shape[1], 3)
        ys, _, _ = run_gpu("drm19", 22, y0[:, sub], 1e-5, 1e-6, 1e-10, rho=rho[sub], F=F[:, sub], kernel=kernel)
        assert np.array_equal(ys, yall[:, sub])


def test_full_size_c3_sampled(oracle):
    """C3 at its BASELINE size (64^3 cells), launch configuration as in bench.py; parity on a
    stratified sample of cells the oracle integrates one by one."""
    mech, n = MECH["h2"]
    y0, rho, F, prog = flame_field(mech, 64, dt=1e-5)
    yg, sg, st = run_gpu("h2", n, y0, 1e-5, 1e-6, 1e-10, rho=rho, F=F)
    G = st["group"]
    assert st["n_failed"] == 0 and st["n_cells"] == 64 ** 3
    idx = stratified_sample(prog, 4000)
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, 1e-5, 1e-6, 1e-10, rho=rho, fext_yc=F,
                                    group=G, threads=8, cells=idx)
    end_state_check(yg[:, idx], yo, 1e-6, 1e-10)


# ------------------------------------------------------------------ global-norm mode (row a12)
@pytest.mark.parametrize("name,L,dt", [("h2", 4, 1e-5), ("drm19", 4, 1e-6), ("drm19", 8, 1e-5), ("gri53", 8, 1e-6)])
def test_global_norm_mode_parity(oracle, name, L, dt):
    """The paper's lockstep batch: one h, q for all cells, batch-wide WRMS (R14, R15 order:
    per-cell sums, 256-cell block partials in order).  GPU (host control loop + device kernels)
    vs the oracle's global-norm variant on identical inputs."""
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, L, dt=dt)
    N = y0.shape[1]
    b = P.Batch(N, n, 1e-6, 1e-10, mode=P.MODE_GLOBAL_NORM)
    b.set_model(name)
    cs = b.attach_cell_stats()
    y = cu(y0)
    b.integrate(0.0, dt, y, f_ext=cu(F), aux=cu(rho))
    st = b.stats()
    yo, so = oracle.integrate_global(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho, fext_yc=F)
    assert so["status"] == 0 and st["n_failed"] == 0
    print(f"global {name} N={N}: gpu nst={st['nst']} nfe={st['nfe']} | oracle nst={so['nst']} nfe={so['nfe']}")
    assert st["nst"] == so["nst"] and st["nfe"] == so["nfe"] and st["netf"] == so["netf"]
    end_state_check(y.cpu().numpy(), yo, 1e-6, 1e-10)
    assert np.all(cs["nst"].cpu().numpy() == so["nst"])


def test_global_norm_nccl_exchange_single_rank(oracle):
    """bdfb_set_comm with nranks = 1: the library's NCCL communicator is created and every batch norm goes
    through the rank-ordered ncclAllGather exchange; with one rank the rank-ordered sum
    is 0 + S, so the run is bit-identical to the run without a communicator."""
    mech, n = MECH["drm19"]
    y0, rho, F, prog = flame_field(mech, 4, dt=1e-6)
    N = y0.shape[1]
    out = []
    for comm in (False, True):
        b = P.Batch(N, n, 1e-6, 1e-10, mode=P.MODE_GLOBAL_NORM)
        b.set_model("drm19")
        if comm:
            b.set_comm(torch.cuda.nccl.unique_id(), 1, 0, N)
        y = cu(y0)
        b.integrate(0.0, 1e-6, y, f_ext=cu(F), aux=cu(rho))
        out.append((y.cpu().numpy(), b.stats()))
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1]["nst"] == out[1][1]["nst"] and out[0][1]["nfe"] == out[1][1]["nfe"]


def test_full_size_c4_sampled(oracle):
    """C4 at its BASELINE size (256^3 = 16.7M DRM19-class cells) in exactly the launch configuration bench.py
    times (the default per-cell kernel); end-state parity on the SURVEY §8(d).3 stratified 65,536-cell sample
    (equal quotas of fresh, reacting and burnt cells) that the oracle integrates cell by cell, plus the
    conservation checks (sum_k Y_k and element sums, F_Y = 0) on every cell.  Reports the identical-stats
    fraction, the |dy|/tol distribution and the number of cells outside the bar (decision flips) to
    gpurun_out/c4_parity_report.json."""
    import json
    import os
    import time
    mech, n = MECH["drm19"]
    y0, rho, F, prog = flame_field(mech, 256, dt=1e-5)
    yg, sg, st = run_gpu("drm19", n, y0, 1e-5, 1e-6, 1e-10, rho=rho, F=F)
    assert st["n_failed"] == 0 and st["n_cells"] == 256 ** 3
    s0 = y0[:-1].sum(axis=0)
    assert np.abs(yg[:-1].sum(axis=0) - s0).max() <= 1e-13
    els, E = element_matrix(mech)
    for j in range(len(els)):     # element sums on every cell (row by row to bound host memory)
        e0 = E[j] @ y0[:-1]
        assert np.all(np.abs(E[j] @ yg[:-1] - e0) <= 1e-13 * (np.abs(E[j]) @ np.abs(y0[:-1]))), els[j]
    idx = stratified_sample(prog, 65536 // 3)
    t0 = time.time()
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0[:, idx], 0.0, 1e-5, 1e-6, 1e-10, rho=rho[idx],
                                    fext_yc=F[:, idx], group=st["group"], threads=os.cpu_count() or 8)
    t_orc = time.time() - t0
    tol = 10.0 * (1e-6 * np.abs(yo) + 1e-10)
    ratio = (np.abs(yg[:, idx] - yo) / tol).max(axis=0)
    same = np.ones(len(idx), bool)
    for k in STAT_KEYS:
        same &= sg[k][idx] == so[k]
    rep = {"cells": int(len(idx)), "identical_stats_fraction": float(same.mean()),
           "outside_bar": int((ratio > 1.0).sum()), "max_ratio": float(ratio.max()),
           "ratio_quantiles": {q: float(np.quantile(ratio, float(q))) for q in ("0.5", "0.9", "0.99", "0.999")},
           "ratio_histogram_log10": np.histogram(np.log10(np.maximum(ratio, 1e-20)), bins=np.arange(-20, 2))[0].tolist(),
           "oracle_seconds": t_orc, "oracle_threads": os.cpu_count()}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/c4_parity_report.json", "w") as f:
        json.dump(rep, f, indent=1)
    print("C4 65536-cell parity:", rep)
    assert np.array_equal(sg["status"][idx], so["status"])
    end_state_check(yg[:, idx], yo, 1e-6, 1e-10)


def test_full_size_c2_sampled(oracle):
    """C2 at its BASELINE size (128^3 Nyx cells, n = 1) as bench.py launches it; parity on sampled cells."""
    e, rho, fe = nyx_field(128)
    dt = 3e15
    yg, sg, st = run_gpu("nyx_kwh", 1, e, dt, 1e-6, 1e-10, rho=rho, F=fe)
    assert st["n_cells"] == 128 ** 3
    idx = np.sort(np.random.default_rng(7).choice(128 ** 3, 20000, replace=False))
    yo, so = oracle.integrate_batch(oracle.Model.nyx_kwh(), e[:, idx], 0.0, dt, 1e-6, 1e-10, rho=rho[idx],
                                    fext_yc=fe[:, idx], threads=8)
    assert np.array_equal(sg["status"][idx], so["status"])
    ok = so["status"] == 0
    end_state_check(yg[:, idx][:, ok], yo[:, ok], 1e-6, 1e-10)


# ------------------------------------------------------------------ typical-value tolerances (Eq. 7, row f2)
@pytest.mark.parametrize("layout", ["YC", "CY"])
def test_typical_values_bitwise(oracle, layout):
    """bdfb_minmax + bdfb_set_atol_typical vs orc_typical_values / orc_atol_from_typical on identical inputs:
    bit-identical (min/max are exact; the midpoint and eta*tv are single roundings on both sides), including
    a ragged cell count and NaN entries (skipped by fmin/fmax on both sides)."""
    y, rho, F, prog = flame_field("drm19_class", 16, dt=1e-5)
    y = y[:, :4093].copy()                                  # ragged
    y[3, 17] = np.nan
    y[0, 4000] = -2.5                                       # a negative entry (signed min/max)
    n, N = y.shape
    b = P.Batch(N, n, 1e-6, 1e-10)
    b.set_model("drm19")
    yd = cu(y if layout == "YC" else y.T)
    tv = b.set_typical_atol(yd, eta=1e-10, floor=1e-30, layout=layout).cpu().numpy()
    tvo = oracle.typical_values(y)
    assert np.array_equal(tv, tvo)
    lo, hi = b.minmax(yd, layout=layout)
    assert np.array_equal(lo.cpu().numpy(), np.fmin.reduce(y, axis=1))
    assert np.array_equal(hi.cpu().numpy(), np.fmax.reduce(y, axis=1))


@pytest.mark.parametrize("name", ["h2", "drm19"])
def test_integrate_with_typical_atol(oracle, name):
    """Integration with the Eq. 7 tolerances (Pele's eta = 1e-10) set on the device (SPLIT kernel) vs the
    oracle with the oracle's own Eq. 7 atol vector: the end states agree within 10 (rtol |y| + atol_i).
    (At looser eta, e.g. 1e-8, single ignition cells can drift past that bar: the two valid trajectories differ
    by the global error -- measured 1 cell of 4096 at ratio 1.12 for H2, exp/tv_check.py.)"""
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 16, dt=1e-5)
    N = y0.shape[1]
    eta = 1e-10
    b = P.Batch(N, n, 1e-6, 1e-10)
    b.set_model(name)
    yd = cu(y0)
    b.set_typical_atol(yd, eta=eta)
    b.integrate(0.0, 1e-5, yd, f_ext=cu(F), aux=cu(rho))
    st = b.stats()
    atol = oracle.atol_from_typical(oracle.typical_values(y0), eta, 1e-30)
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, 1e-5, 1e-6, atol, rho=rho, fext_yc=F,
                                    group=b.wrms_group, threads=8)
    assert st["n_failed"] == 0 and np.all(so["status"] == 0)
    yg = yd.cpu().numpy()
    tol = 10.0 * (1e-6 * np.abs(yo) + atol[:, None])
    assert np.all(np.abs(yg - yo) <= tol)


# ------------------------------------------------------------------ difference-quotient Jacobian (row f1)
@pytest.mark.parametrize("name", ["h2", "drm19"])
def test_dq_jacobian_parity(oracle, name):
    """SPLIT kernel with the difference-quotient Jacobian (bdfb_set_jacobian DQ; approaches 3A/3B)
    vs the oracle's orc_jac_dq path on identical inputs: end states within 10 (rtol |y| + atol); and vs the
    oracle's analytic-Jacobian run within 100 rtol (SPEC AC8)."""
    mech, n = MECH[name]
    y0, rho, F, prog = flame_field(mech, 16, dt=1e-5)
    b = P.Batch(y0.shape[1], n, 1e-6, 1e-10)
    b.set_model(name)
    b.set_jacobian("dq")
    cs = b.attach_cell_stats()
    y = cu(y0)
    b.integrate(0.0, 1e-5, y, f_ext=cu(F), aux=cu(rho))
    st = b.stats()
    assert st["n_failed"] == 0
    yg = y.cpu().numpy()
    m = oracle.Model.mechanism(mech)
    yo, so = oracle.integrate_batch(m, y0, 0.0, 1e-5, 1e-6, 1e-10, rho=rho, fext_yc=F, group=b.wrms_group, threads=8,
                                    ls=oracle.LS_DENSE_DQ)
    end_state_check(yg, yo, 1e-6, 1e-10)
    ya, _ = oracle.integrate_batch(m, y0, 0.0, 1e-5, 1e-6, 1e-10, rho=rho, fext_yc=F, group=b.wrms_group, threads=8)
    assert np.all(np.abs(yg - ya) <= 100 * 1e-6 * np.abs(ya) + 1e-9)
    same = np.mean([all(cs[k].cpu().numpy()[c] == so[k][c] for k in STAT_KEYS) for c in range(y0.shape[1])])
    print(f"{name} DQ: identical per-cell stats vs the oracle's DQ run {same:.4f}")


def test_dq_jacobian_unsupported_paths():
    """DQ is offered only by the SPLIT mechanism kernel in per-cell mode."""
    b = P.Batch(64, 10, 1e-6, 1e-10)
    b.set_kernel("thread")
    b.set_model("h2")
    with pytest.raises(RuntimeError):
        b.set_jacobian("dq")
    b2 = P.Batch(64, 3, 1e-6, 1e-10)
    b2.set_model("robertson")
    with pytest.raises(RuntimeError):
        b2.set_jacobian("dq")


# ------------------------------------------------------------------ auto-ignition box
@pytest.mark.parametrize("name,dt", [("h2", 1e-4), ("drm19", 1e-3)])
def test_autoignition_box_parity(oracle, name, dt):
    """The paper's batched-solver test workload: a uniform mixture with T rising along x, so part of the
    domain ignites within the step (the stiffest cells of the batch): SPLIT kernel vs the oracle within
    10 (rtol |y| + atol) per cell and component, identical statuses, sum_k Y_k conserved on both sides."""
    from synth import autoignition_box
    mech, n = MECH[name]
    y0, rho = autoignition_box(mech, 16)
    yg, sg, st = run_gpu(name, n, y0, dt, 1e-6, 1e-10, rho=rho)
    yo, so = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho,
                                    group=st["group"], threads=8)
    assert np.array_equal(sg["status"], so["status"]) and st["n_failed"] == 0
    end_state_check(yg, yo, 1e-6, 1e-10)
    yp, _ = oracle.integrate_batch(oracle.Model.mechanism(mech), y0, 0.0, dt, 1e-6, 1e-10, rho=rho,
                                   group=st["group"], threads=8, plain=True)
    end_state_check(yg, yp, 1e-6, 1e-10)
    rise = yg[-1] - y0[-1]
    assert np.mean(rise > 100.0) > 0.05 and np.mean(rise < 100.0) > 0.05, "the step must straddle ignition"
    s0 = y0[:-1].sum(axis=0)
    assert np.abs(yg[:-1].sum(axis=0) - s0).max() <= 1e-12 and np.abs(yo[:-1].sum(axis=0) - s0).max() <= 1e-12
