"""Counter-based seeded fields (see synth/__init__.py)."""
from __future__ import annotations

import json
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SEED_BASE = 2405017130          # seed S = 2405017130 + config
RU = 8.31446261815324e7         # erg/(mol K)  (ideal-gas density of the initial mixture)
PATM = 1013250.0

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def config_seed(c: int) -> int:
    return SEED_BASE + int(c)


def splitmix64(x):
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _key(seed, cells, field):
    cells = np.asarray(cells, dtype=np.uint64)
    with np.errstate(over="ignore"):
        k = splitmix64(np.uint64(seed) * np.uint64(0x100000001B3) + np.uint64(field))
        return splitmix64(k ^ (cells * np.uint64(0xD1B54A32D192ED03)))


def uniform(seed, cells, field):
    """U[0,1) per (seed, cell, field): 53-bit mantissa from SplitMix64."""
    return (_key(seed, cells, field) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def gaussian(seed, cells, field):
    """N(0,1) per (seed, cell, field) by Box-Muller on two keyed uniforms."""
    u1 = uniform(seed, cells, 2 * field + 1000)
    u2 = uniform(seed, cells, 2 * field + 1001)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def grid_xyz(L, cells):
    c = np.asarray(cells, dtype=np.int64)
    i = c % L
    j = (c // L) % L
    k = c // (L * L)
    return (i + 0.5) / L, (j + 0.5) / L, (k + 0.5) / L


def fourier_field(seed, field, L, cells, modes=16, kmax=4):
    """Unit-variance smooth field: sum_m a_m cos(2 pi k_m.x + theta_m), integer |k_m| in [1, kmax]."""
    x, y, z = grid_xyz(L, cells)
    out = np.zeros(len(np.atleast_1d(cells)))
    m = np.arange(modes, dtype=np.uint64)
    ks = []
    for d in range(3):
        ks.append(np.floor(uniform(seed, m, 5000 + 10 * field + d) * (2 * kmax + 1)).astype(np.int64) - kmax)
    amp = gaussian(seed, m, 6000 + field) / 4.0
    th = 2 * np.pi * uniform(seed, m, 7000 + field)
    var = 0.0
    for i in range(modes):
        kv = np.array([ks[0][i], ks[1][i], ks[2][i]])
        if not np.any(kv):
            kv[0] = 1
        out += amp[i] * np.cos(2 * np.pi * (kv[0] * x + kv[1] * y + kv[2] * z) + th[i])
        var += amp[i] ** 2 / 2
    return out / math.sqrt(var)


# ---------------------------------------------------------------- C1 Robertson
def robertson_field(N, seed=None, cells=None):
    """cell 0 = (1,0,0); cells c>=1: a=3e-5 u1, b=0.5 u2, y0=(1-a-b, a, b). YC [3, M]."""
    seed = config_seed(1) if seed is None else seed
    c = np.arange(N) if cells is None else np.asarray(cells)
    a = 3e-5 * uniform(seed, c, 1)
    b = 0.5 * uniform(seed, c, 2)
    y = np.stack([1.0 - a - b, a, b])
    y[:, c == 0] = np.array([[1.0], [0.0], [0.0]])
    return y


# ---------------------------------------------------------------- C2 Nyx
NYX_RHO_MEAN = 2.69e-29         # g/cm^3, Omega_b h^2 = 0.0224 at z = 3
NYX_DT = 3.0e15                 # s (~95 Myr), calibrated so 10-30% of cells cool within dt


def nyx_field(L, seed=None, cells=None, dt=NYX_DT):
    """SURVEY §8(d).1 C2 on an L^3 grid: returns (e [1, M], rho [M], F_e [1, M])."""
    seed = config_seed(2) if seed is None else seed
    c = np.arange(L ** 3) if cells is None else np.asarray(cells)
    G = fourier_field(seed, 1, L, c)
    sigma = 1.5
    delta = np.exp(sigma * G - sigma ** 2 / 2)
    rho = delta * NYX_RHO_MEAN
    T = 1e4 * delta ** 0.6 * 10.0 ** (0.1 * gaussian(seed, c, 3))
    shocked = uniform(seed, c, 4) < 0.05
    T = np.where(shocked, 10.0 ** (5.0 + 2.0 * uniform(seed, c, 5)), T)
    mp, kB = 1.67262192369e-24, 1.380649e-16
    e = T * kB / ((5.0 / 3.0 - 1.0) * 0.59 * mp)
    fe = 0.1 * e * gaussian(seed, c, 6) / dt
    return e[None, :], rho, fe[None, :]


# ---------------------------------------------------------------- C3/C4 flames
MIXTURES = {
    "h2_lidryer": ({"H2": 0.02852, "O2": 0.22635, "N2": 0.74513}, 700.0, 1100.0),
    "drm19_class": ({"CH4": 0.05519, "O2": 0.22015, "N2": 0.72466}, 700.0, 1400.0),
    "gri53_class": ({"CH4": 0.05519, "O2": 0.22015, "N2": 0.72466}, 700.0, 1400.0),   # C5: CH4/air as C4
}
MECH_CONFIG = {"h2_lidryer": 3, "drm19_class": 4, "gri53_class": 5}   # seed S = 2405017130 + config
DELTA_FLAME = 0.0971            # tanh width: ~15% of cells with 0.02 < c < 0.98 (unit-variance phi)


def load_table(mech):
    with open(os.path.join(REPO, "mechanisms", mech + ".json")) as f:
        return json.load(f)


def load_trajectory(mech):
    path = os.path.join(HERE, "data", f"{mech}_trajectory.npz")
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run python synth/make_trajectories.py")
    d = np.load(path)
    return d["c"], d["states"], float(d["rho"])


def fresh_state(mech):
    tab = load_table(mech)
    sp = [s["name"] for s in tab["species"]]
    W = np.array([s["W"] for s in tab["species"]])
    fr, T_cold, T_u = MIXTURES[mech]
    Y = np.zeros(len(sp))
    for k, v in fr.items():
        Y[sp.index(k)] = v
    Y /= Y.sum()
    rho_u = PATM / (RU * T_u * np.sum(Y / W))
    return Y, W, T_cold, T_u, rho_u


def flame_field(mech, L, seed=None, cells=None, dt=1e-5, forcing=True, threads=None, chunk=1 << 19):
    """SURVEY §8(d).1 flame-field template: returns (y [n, M] YC, rho [M], F [n, M], c [M]).
    Large requests are generated in cell chunks on a thread pool (values are per-cell pure
    functions, so chunking does not change them)."""
    c_idx = np.arange(L ** 3) if cells is None else np.asarray(cells)
    M = len(c_idx)
    if M > chunk:
        from concurrent.futures import ThreadPoolExecutor
        K = len(fresh_state(mech)[0])
        y = np.empty((K + 1, M))
        F = np.empty((K + 1, M))
        rho = np.empty(M)
        prog = np.empty(M)
        def work(s):
            e = min(M, s + chunk)
            y[:, s:e], rho[s:e], F[:, s:e], prog[s:e] = flame_field(mech, L, seed, c_idx[s:e], dt, forcing,
                                                                    chunk=chunk)
        with ThreadPoolExecutor(max_workers=threads or min(32, os.cpu_count() or 1)) as ex:
            list(ex.map(work, range(0, M, chunk)))
        return y, rho, F, prog
    return _flame_chunk(mech, L, seed, c_idx, dt, forcing)


def _flame_chunk(mech, L, seed, c_idx, dt, forcing):
    seed = config_seed(MECH_CONFIG[mech]) if seed is None else seed
    M = len(c_idx)
    Yf, W, T_cold, T_u, rho_u = fresh_state(mech)
    K = len(Yf)
    cgrid, states, rho_traj = load_trajectory(mech)        # states [P, K+1], cgrid [P] increasing
    phi = fourier_field(seed, 1, L, c_idx)
    prog = 0.5 * (1.0 + np.tanh(phi / DELTA_FLAME))
    y = np.empty((K + 1, M))
    for k in range(K + 1):
        y[k] = np.interp(prog, cgrid, states[:, k])
    fresh = prog < 0.02
    burnt = prog > 0.98
    y[:K, fresh] = Yf[:, None]
    y[K, fresh] = T_cold
    y[:, burnt] = states[-1][:, None]
    # jitter
    y[K] *= 1.0 + 0.005 * gaussian(seed, c_idx, 10)
    for k in range(K):
        if np.any(y[k] != 0):
            y[k] *= 1.0 + 0.01 * gaussian(seed, c_idx, 100 + k)
    y[:K] = np.maximum(y[:K], 0.0)
    y[:K] /= y[:K].sum(axis=0, keepdims=True)
    rho = np.where(fresh, rho_u * T_u / T_cold, rho_traj) * (1.0 + 0.01 * gaussian(seed, c_idx, 11))
    F = np.zeros_like(y)
    if forcing:
        F[K] = (5.0 / dt) * gaussian(seed, c_idx, 12)
    return y, rho, F, prog


def stratified_sample(prog, per_class, seed=0):
    """Indices with equal quotas of fresh (c<0.02), reacting and burnt (c>0.98) cells."""
    cls = [np.where(prog < 0.02)[0], np.where((prog >= 0.02) & (prog <= 0.98))[0], np.where(prog > 0.98)[0]]
    out = []
    for j, ix in enumerate(cls):
        if len(ix) == 0:
            continue
        u = uniform(seed, ix, 900 + j)
        out.append(ix[np.argsort(u)[:per_class]])
    return np.sort(np.concatenate(out))


# ---------------------------------------------------------------- auto-ignition box
AUTOIGNITION_T = {"h2_lidryer": (900.0, 1300.0), "drm19_class": (1200.0, 1700.0), "gri53_class": (1200.0, 1700.0)}


def autoignition_box(mech, L, cells=None):
    """SURVEY §8(d).1 second workload (the paper's batched-solver test): a uniform fresh mixture at
    1 atm with T rising linearly along x (H2: 900 -> 1300 K; CH4: 1200 -> 1700 K), so part of the domain
    ignites within the step.  Returns (y [n, M] YC, rho [M]); no forcing."""
    c_idx = np.arange(L ** 3) if cells is None else np.asarray(cells)
    Yf, W, T_cold, T_u, rho_u = fresh_state(mech)
    x, _, _ = grid_xyz(L, c_idx)
    t0, t1 = AUTOIGNITION_T[mech]
    T = t0 + (t1 - t0) * (x - 0.5 / L) / (1.0 - 1.0 / L)
    y = np.empty((len(Yf) + 1, len(c_idx)))
    y[:-1] = Yf[:, None]
    y[-1] = T
    rho = PATM / (RU * T * np.sum(Yf / W))
    return y, rho
