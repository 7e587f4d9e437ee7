"""ctypes wrapper of the C oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
(paper_2405_01713_b200).  It shares no code with the CUDA path; it reads the
mechanism JSON tables (problem data) itself.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "liboracle.so")

MODEL_LINEAR, MODEL_ROBERTSON, MODEL_KWH, MODEL_MECH = 0, 1, 2, 3
LS_DENSE, LS_DIAG, LS_DENSE_DQ, LS_GMRES = 0, 1, 2, 3
METHOD_BDF, METHOD_ERK4 = 0, 1
STATUS = {0: "OK", 1: "TOO_MUCH_WORK", 2: "ERR_FAILURE", 3: "CONV_FAILURE", 4: "RHS_FAIL",
          5: "NONFINITE_INPUT"}
QMAX = 5


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, f) for f in ("bdf.c", "linalg.c", "models.c", "krylov.c", "erk.c",
                                              "oracle.h", "mech_body.h")]
    if force or not os.path.exists(LIB_PATH) or any(
            os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in srcs):
        subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
    return LIB_PATH


class KwhParams(C.Structure):
    _fields_ = [("z", C.c_double), ("X", C.c_double), ("Y", C.c_double), ("gamma_ad", C.c_double),
                ("gph", C.c_double * 3), ("eph", C.c_double * 3)]


class Mech(C.Structure):
    _fields_ = [("K", C.c_int), ("nr", C.c_int), ("W", C.POINTER(C.c_double)),
                ("nasa", C.POINTER(C.c_double)), ("reac", C.POINTER(C.c_int)),
                ("prod", C.POINTER(C.c_int)), ("rev", C.POINTER(C.c_int)),
                ("type", C.POINTER(C.c_int)), ("arr", C.POINTER(C.c_double)),
                ("arr0", C.POINTER(C.c_double)), ("troe", C.POINTER(C.c_double)),
                ("has_t2", C.POINTER(C.c_int)), ("eff", C.POINTER(C.c_double))]


class Problem(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int), ("lam", C.POINTER(C.c_double)),
                ("rob_k", C.POINTER(C.c_double)), ("kwh", C.POINTER(KwhParams)),
                ("mech", C.POINTER(Mech)), ("rho", C.c_double), ("fext", C.POINTER(C.c_double))]


class Opts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.POINTER(C.c_double)), ("qmax", C.c_int),
                ("mxstep", C.c_int64), ("h0", C.c_double), ("hmin", C.c_double), ("hmax", C.c_double),
                ("ls", C.c_int), ("group", C.c_int), ("method", C.c_int), ("maxl", C.c_int),
                ("plain", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("status", C.c_int32), ("nst", C.c_int32), ("nfe", C.c_int32), ("nje", C.c_int32),
                ("nsetups", C.c_int32), ("nni", C.c_int32), ("netf", C.c_int32), ("ncfn", C.c_int32),
                ("q_last", C.c_int32), ("h_last", C.c_double), ("t_reached", C.c_double), ("nli", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Trace(C.Structure):
    _fields_ = [("cap", C.c_int), ("count", C.c_int), ("tn", C.POINTER(C.c_double)),
                ("h", C.POINTER(C.c_double)), ("q", C.POINTER(C.c_int)), ("zn", C.POINTER(C.c_double))]


ATIMES = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))
GMRES_STATUS = {0: "SUCCESS", 1: "RES_REDUCED", 2: "CONV_FAIL", 3: "ATIMES_FAIL_REC", 4: "QRFACT_FAIL",
                5: "QRSOL_FAIL", -1: "ATIMES_FAIL_UNREC"}

_lib = None
_lock = threading.Lock()


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(LIB_PATH)
            dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
            L.orc_wrms.restype = C.c_double
            L.orc_wrms.argtypes = [C.c_int, dp, dp, C.c_int]
            L.orc_jac_dq.restype = C.c_int
            L.orc_jac_dq.argtypes = [C.POINTER(Problem), C.c_double, dp, dp, dp, C.c_double, dp]
            L.orc_typical_values.restype = None
            L.orc_typical_values.argtypes = [C.c_int, C.c_int64, dp, dp]
            L.orc_atol_from_typical.restype = None
            L.orc_atol_from_typical.argtypes = [C.c_int, dp, C.c_double, C.c_double, dp]
            L.orc_lu_factor.restype = C.c_int
            L.orc_lu_factor.argtypes = [C.c_int, dp, ip]
            L.orc_lu_solve.restype = None
            L.orc_lu_solve.argtypes = [C.c_int, dp, ip, dp]
            L.orc_lu_solve_div.restype = None
            L.orc_lu_solve_div.argtypes = [C.c_int, dp, ip, dp]
            L.orc_choose_eta.restype = C.c_double
            L.orc_choose_eta.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_int, C.c_double, C.c_int,
                                         C.POINTER(C.c_int), dp]
            L.orc_newton_once.restype = C.c_int
            L.orc_newton_once.argtypes = [C.POINTER(Problem), C.POINTER(Opts), C.c_double, C.c_double,
                                          C.c_double, C.c_double, dp, dp, dp, dp, dp, C.POINTER(C.c_int),
                                          C.POINTER(C.c_int)]
            L.orc_gmres.restype = C.c_int
            L.orc_gmres.argtypes = [C.c_int, C.c_int, ATIMES, C.c_void_p, dp, dp, dp, C.c_double, dp,
                                    C.POINTER(C.c_int), dp]
            L.orc_erk_step.restype = C.c_int
            L.orc_erk_step.argtypes = [C.POINTER(Problem), C.c_double, C.c_double, dp, dp, dp, dp,
                                       C.POINTER(C.c_int)]
            L.orc_integrate_erk.restype = C.c_int
            L.orc_integrate_erk.argtypes = [C.POINTER(Problem), C.POINTER(Opts), C.c_double, C.c_double, dp,
                                            C.POINTER(Stats)]
            L.orc_rhs.restype = C.c_int
            L.orc_rhs.argtypes = [C.POINTER(Problem), C.c_double, dp, dp]
            L.orc_rhs_scale.restype = C.c_int
            L.orc_rhs_scale.argtypes = [C.POINTER(Problem), C.c_double, dp, dp]
            L.orc_jac.restype = C.c_int
            L.orc_jac.argtypes = [C.POINTER(Problem), C.c_double, dp, dp]
            L.orc_kwh_state.restype = C.c_int
            L.orc_kwh_state.argtypes = [C.POINTER(Problem), C.c_double, dp]
            L.orc_root.restype = C.c_double
            L.orc_root.argtypes = [C.c_double, C.c_int]
            L.orc_set_bdf.restype = None
            L.orc_set_bdf.argtypes = [C.c_int, C.c_double, dp, C.c_int, dp, dp]
            L.orc_integrate.restype = C.c_int
            L.orc_integrate.argtypes = [C.POINTER(Problem), C.POINTER(Opts), C.c_double, C.c_double, dp,
                                        C.POINTER(Stats), C.POINTER(Trace)]
            L.orc_integrate_global.restype = C.c_int
            L.orc_integrate_global.argtypes = [C.POINTER(Problem), C.POINTER(Opts), C.c_double, C.c_double,
                                               C.c_int64, dp, dp, dp, C.POINTER(Stats)]
            L.orc_integrate_batch.restype = None
            L.orc_integrate_batch.argtypes = [C.POINTER(Problem), C.POINTER(Opts), C.c_double, C.c_double,
                                              C.c_int64, C.c_int64, C.c_int64, dp, dp, dp, C.POINTER(Stats)]
            _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


# ---- primitives ---------------------------------------------------------------
def wrms(v, w, group=1):
    v = np.ascontiguousarray(v, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    return lib().orc_wrms(len(v), _dp(v), _dp(w), int(group))


def typical_values(y_yc):
    """Eq. 7 typical values of a YC field y[n, N] (orc_typical_values)."""
    y = np.ascontiguousarray(y_yc, dtype=np.float64)
    n, N = y.shape
    tv = np.empty(n)
    lib().orc_typical_values(n, N, _dp(y), _dp(tv))
    return tv


def atol_from_typical(tv, eta=1e-10, floor=1e-30):
    """Eq. 7: atol_i = max(eta tv_i, floor) (orc_atol_from_typical)."""
    tv = np.ascontiguousarray(tv, dtype=np.float64)
    out = np.empty(len(tv))
    lib().orc_atol_from_typical(len(tv), _dp(tv), float(eta), float(floor), _dp(out))
    return out


def lu_factor(M):
    M = np.array(M, dtype=np.float64, order="C", copy=True)
    n = M.shape[0]
    piv = np.zeros(n, dtype=np.int32)
    info = lib().orc_lu_factor(n, _dp(M), _ip(piv))
    return M, piv, info


def lu_solve(LU, piv, b, plain=False):
    """LU_SOLVE: reciprocal-multiply back substitution (R16), or true division when plain."""
    LU = np.ascontiguousarray(LU, dtype=np.float64)
    piv = np.ascontiguousarray(piv, dtype=np.int32)
    b = np.array(b, dtype=np.float64, copy=True)
    (lib().orc_lu_solve_div if plain else lib().orc_lu_solve)(LU.shape[0], _dp(LU), _ip(piv), _dp(b))
    return b


def choose_eta(q, qwait, dsm, ddn=0.0, dup=None, etamax=10.0, h=1.0, hmax=0.0, plain=False):
    """PREPARE_NEXT scalar part (orc_choose_eta): returns (eta, qprime, hprime, qwait_out)."""
    qw = C.c_int(int(qwait))
    qp = C.c_int(0)
    hp = C.c_double(0.0)
    eta = lib().orc_choose_eta(int(q), C.byref(qw), float(etamax), float(h), float(hmax), float(dsm), float(ddn),
                               0 if dup is None else 1, 0.0 if dup is None else float(dup), int(plain),
                               C.byref(qp), C.byref(hp))
    return eta, qp.value, hp.value, qw.value


def newton_once(model, zn0, zn1, ewt, h, rl1, tol, rho=1.0, fext=None, tn=0.0, atol=1e-10, rtol=1e-6):
    """One NEWTON solve of the listing with a forced matrix setup (orc_newton_once).
    Returns (status, acor, acnrm, nni, nfe)."""
    zn0 = np.ascontiguousarray(zn0, dtype=np.float64)
    zn1 = np.ascontiguousarray(zn1, dtype=np.float64)
    ewt = np.ascontiguousarray(ewt, dtype=np.float64)
    p = model.problem(rho, fext)
    o = make_opts(model.n, rtol, atol, ls=LS_DENSE)
    acor = np.zeros(model.n)
    acn = C.c_double(0.0)
    nni, nfe = C.c_int(0), C.c_int(0)
    r = lib().orc_newton_once(C.byref(p), C.byref(o), float(tn), float(h), float(rl1), float(tol), _dp(zn0),
                              _dp(zn1), _dp(ewt), _dp(acor), C.byref(acn), C.byref(nni), C.byref(nfe))
    return r, acor, acn.value, nni.value, nfe.value


def gmres(A, b, s1=None, s2=None, delta=0.0, maxl=None):
    """Scaled GMRES of the oracle (orc_gmres, Eq. 5-6) on a dense matrix A or a callable v -> A v.
    Returns (x, status, iterations, rotation residual)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = len(b)
    Am = None if callable(A) else np.asarray(A, dtype=np.float64)

    def _at(ctx, v, z):
        vv = np.ctypeslib.as_array(v, shape=(n,)).copy()
        zz = A(vv) if Am is None else Am @ vv
        for i in range(n):
            z[i] = float(zz[i])
        return 0

    cb = ATIMES(_at)
    x = np.zeros(n)
    it = C.c_int(0)
    rn = C.c_double(0.0)
    s1a = None if s1 is None else np.ascontiguousarray(s1, dtype=np.float64)
    s2a = None if s2 is None else np.ascontiguousarray(s2, dtype=np.float64)
    r = lib().orc_gmres(n, int(maxl or n), cb, None, _dp(b), _dp(s1a) if s1a is not None else None,
                        _dp(s2a) if s2a is not None else None, float(delta), _dp(x), C.byref(it), C.byref(rn))
    return x, r, it.value, rn.value


def erk_step(model, y, h, rho=1.0, fext=None, t=0.0):
    """One step of the embedded 4(3) pair (orc_erk_step): returns (ynew, err, status, nfe)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    yn = np.zeros(model.n)
    er = np.zeros(model.n)
    nfe = C.c_int(0)
    p = model.problem(rho, fext)
    r = lib().orc_erk_step(C.byref(p), float(t), float(h), _dp(y), None, _dp(yn), _dp(er), C.byref(nfe))
    return yn, er, r, nfe.value


def root(x, L):
    return lib().orc_root(float(x), int(L))


def set_bdf(q, h, tau, qwait):
    tau7 = np.zeros(7)
    tau7[1:1 + len(tau)] = tau
    l = np.zeros(QMAX + 1)
    tq = np.zeros(6)
    lib().orc_set_bdf(int(q), float(h), _dp(tau7), int(qwait), _dp(l), _dp(tq))
    return l, tq


# ---- models -------------------------------------------------------------------
def load_mech_table(name_or_path):
    path = name_or_path
    if not os.path.exists(path):
        path = os.path.join(REPO, "mechanisms", name_or_path + ".json")
    with open(path) as f:
        return json.load(f)


class MechData:
    """The oracle's own flattening of a mechanism table into orc_mech arrays."""

    TYPES = {"elementary": 0, "three_body": 1, "lindemann": 2, "troe": 3}

    def __init__(self, table):
        sp = [s["name"] for s in table["species"]]
        idx = {s: i for i, s in enumerate(sp)}
        K, I = len(sp), len(table["reactions"])
        self.table, self.K, self.nr, self.species = table, K, I, sp
        self.W = np.array([s["W"] for s in table["species"]], dtype=np.float64)
        self.nasa = np.zeros((K, 15))
        for k, s in enumerate(table["species"]):
            self.nasa[k, 0] = s["nasa"]["Tmid"]
            self.nasa[k, 1:8] = s["nasa"]["low"]
            self.nasa[k, 8:15] = s["nasa"]["high"]
        self.reac = -np.ones((I, 3), dtype=np.int32)
        self.prod = -np.ones((I, 3), dtype=np.int32)
        self.rev = np.zeros(I, dtype=np.int32)
        self.type = np.zeros(I, dtype=np.int32)
        self.arr = np.zeros((I, 3))
        self.arr0 = np.ones((I, 3))
        self.troe = np.ones((I, 4))
        self.has_t2 = np.zeros(I, dtype=np.int32)
        self.eff = np.zeros((I, K))
        for r, rx in enumerate(table["reactions"]):
            for s, name in enumerate(rx["reactants"]):
                self.reac[r, s] = idx[name]
            for s, name in enumerate(rx["products"]):
                self.prod[r, s] = idx[name]
            self.rev[r] = 1 if rx["reversible"] else 0
            self.type[r] = self.TYPES[rx["type"]]
            self.arr[r] = (rx["A"], rx["b"], rx["Ea"])
            if "low" in rx:
                self.arr0[r] = (rx["low"]["A"], rx["low"]["b"], rx["low"]["Ea"])
            if "troe" in rx:
                t = rx["troe"]
                self.troe[r, :len(t)] = t
                self.has_t2[r] = 1 if len(t) == 4 else 0
            if "efficiencies" in rx:
                for name, v in rx["efficiencies"].items():
                    self.eff[r, idx[name]] = v
        self.c = Mech(K, I, _dp(self.W), _dp(self.nasa), _ip(self.reac), _ip(self.prod), _ip(self.rev),
                      _ip(self.type), _dp(self.arr), _dp(self.arr0), _dp(self.troe), _ip(self.has_t2),
                      _dp(self.eff))


DEFAULT_KWH = dict(z=3.0, X=0.76, Y=0.24, gamma_ad=5.0 / 3.0, gph=(1.0e-12, 6.0e-13, 3.0e-15),
                   eph=(4.0e-24, 5.0e-24, 7.0e-26))
ROBERTSON_K = (0.04, 3e7, 1e4)


@dataclass
class Model:
    """Problem description (Python side).  kind: 'linear'|'robertson'|'kwh'|<mech name>."""
    kind: str
    n: int = 0
    lam: object = None
    rob_k: tuple = ROBERTSON_K
    kwh: dict = field(default_factory=lambda: dict(DEFAULT_KWH))
    mech: MechData = None

    @staticmethod
    def linear(lam):
        lam = np.atleast_1d(np.asarray(lam, dtype=np.float64))
        return Model("linear", n=len(lam), lam=lam)

    @staticmethod
    def robertson(k=ROBERTSON_K):
        return Model("robertson", n=3, rob_k=tuple(k))

    @staticmethod
    def nyx_kwh(**kw):
        p = dict(DEFAULT_KWH)
        p.update(kw)
        return Model("kwh", n=1, kwh=p)

    @staticmethod
    def mechanism(name):
        md = MechData(load_mech_table(name))
        return Model(name, n=md.K + 1, mech=md)

    def problem(self, rho=1.0, fext=None):
        """Build a C orc_problem; keeps referenced arrays alive on the returned object."""
        keep = []
        p = Problem()
        p.n = self.n
        p.rho = float(rho)
        if self.kind == "linear":
            p.kind = MODEL_LINEAR
            lam = np.ascontiguousarray(self.lam)
            keep.append(lam)
            p.lam = _dp(lam)
        elif self.kind == "robertson":
            p.kind = MODEL_ROBERTSON
            k = np.array(self.rob_k, dtype=np.float64)
            keep.append(k)
            p.rob_k = _dp(k)
        elif self.kind == "kwh":
            p.kind = MODEL_KWH
            q = self.kwh
            kp = KwhParams(q["z"], q["X"], q["Y"], q["gamma_ad"], (C.c_double * 3)(*q["gph"]),
                           (C.c_double * 3)(*q["eph"]))
            keep.append(kp)
            p.kwh = C.pointer(kp)
        else:
            p.kind = MODEL_MECH
            keep.append(self.mech)
            p.mech = C.pointer(self.mech.c)
        if fext is not None:
            fe = np.ascontiguousarray(fext, dtype=np.float64)
            keep.append(fe)
            p.fext = _dp(fe)
        p._keep = keep
        return p

    @property
    def default_ls(self):
        return LS_DIAG if self.kind == "kwh" else LS_DENSE


def rhs(model, y, rho=1.0, fext=None, t=0.0):
    y = np.ascontiguousarray(y, dtype=np.float64)
    f = np.zeros(model.n)
    p = model.problem(rho, fext)
    r = lib().orc_rhs(C.byref(p), t, _dp(y), _dp(f))
    return f, r


def rhs_scale(model, y, rho=1.0, fext=None, t=0.0):
    y = np.ascontiguousarray(y, dtype=np.float64)
    S = np.zeros(model.n)
    p = model.problem(rho, fext)
    r = lib().orc_rhs_scale(C.byref(p), t, _dp(y), _dp(S))
    return S, r


def jac(model, y, rho=1.0, fext=None, t=0.0):
    y = np.ascontiguousarray(y, dtype=np.float64)
    J = np.zeros((model.n, model.n))
    p = model.problem(rho, fext)
    r = lib().orc_jac(C.byref(p), t, _dp(y), _dp(J))
    return J, r


def jac_dq(model, y, fy, ewt, h, rho=1.0, fext=None, t=0.0):
    """Difference-quotient Jacobian (orc_jac_dq, CVODE's cvLsDenseDQJac)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    fy = np.ascontiguousarray(fy, dtype=np.float64)
    ewt = np.ascontiguousarray(ewt, dtype=np.float64)
    J = np.zeros((model.n, model.n))
    p = model.problem(rho, fext)
    r = lib().orc_jac_dq(C.byref(p), t, _dp(y), _dp(fy), _dp(ewt), float(h), _dp(J))
    return J, r


def kwh_state(model, e, rho):
    """Converged KWH ionisation state: dict(T, nH0, nHp, nHe0, nHep, nHepp, ne, g), status."""
    out = np.zeros(8)
    p = model.problem(rho, None)
    r = lib().orc_kwh_state(C.byref(p), float(e), _dp(out))
    return dict(zip(["T", "nH0", "nHp", "nHe0", "nHep", "nHepp", "ne", "g"], out)), r


def make_opts(n, rtol, atol, qmax=5, mxstep=10000, h0=0.0, hmin=0.0, hmax=0.0, ls=LS_DENSE, group=1, plain=False,
              method=METHOD_BDF, maxl=0):
    """plain=True: the listing's plain arithmetic (libm pow roots, true division in LU_SOLVE) instead of
    readings R25/R16 -- the CUDA path must match both within the end-state band."""
    at = np.ascontiguousarray(np.broadcast_to(np.asarray(atol, dtype=np.float64), (n,)))
    o = Opts(rtol, _dp(at), qmax, mxstep, h0, hmin, hmax, ls, group, method, maxl, 1 if plain else 0)
    o._keep = at
    return o


def integrate(model, y0, t0, tf, rtol, atol, rho=1.0, fext=None, trace=0, ls=None, group=1, **kw):
    """Integrate one cell.  Returns (y, stats dict, trace dict or None)."""
    y = np.array(y0, dtype=np.float64, copy=True)
    p = model.problem(rho, fext)
    o = make_opts(model.n, rtol, atol, ls=model.default_ls if ls is None else ls, group=group, **kw)
    st = Stats()
    tr = None
    trp = None
    if trace:
        tr = dict(tn=np.zeros(trace), h=np.zeros(trace), q=np.zeros(trace, dtype=np.int32),
                  zn=np.zeros((trace, QMAX + 1, model.n)))
        trp = Trace(trace, 0, _dp(tr["tn"]), _dp(tr["h"]), _ip(tr["q"]), _dp(tr["zn"]))
    lib().orc_integrate(C.byref(p), C.byref(o), float(t0), float(tf), _dp(y), C.byref(st),
                        C.byref(trp) if trp is not None else None)
    if trp is not None:
        c = trp.count
        tr = {k: v[:c] for k, v in tr.items()}
    return y, st.as_dict(), tr


def integrate_global(model, y_yc, t0, tf, rtol, atol, rho=None, fext_yc=None, group=1, **kw):
    """Global-norm mode (lockstep batch, batch-wide WRMS): returns (y [n, N], stats dict)."""
    y = np.array(y_yc, dtype=np.float64, copy=True, order="C")
    n, N = y.shape
    fe = None if fext_yc is None else np.ascontiguousarray(fext_yc, dtype=np.float64)
    rh = None if rho is None else np.ascontiguousarray(rho, dtype=np.float64)
    p = model.problem(1.0, None)
    o = make_opts(n, rtol, atol, ls=LS_DENSE, group=group, **kw)
    st = Stats()
    lib().orc_integrate_global(C.byref(p), C.byref(o), float(t0), float(tf), N, _dp(y),
                               _dp(fe) if fe is not None else None, _dp(rh) if rh is not None else None,
                               C.byref(st))
    return y, st.as_dict()


STAT_FIELDS = ["status", "nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn", "q_last", "h_last", "t_reached",
               "nli"]


def integrate_batch(model, y_yc, t0, tf, rtol, atol, rho=None, fext_yc=None, ls=None, group=1, threads=1,
                    chunk=16, cells=None, **kw):
    """Integrate cells of a YC field y[k, N] (in place on a copy).

    cells: optional index array (subset); threads: host threads (ctypes releases the GIL).
    Returns (y_out [n, M], stats structured dict of arrays) for the selected cells."""
    y_yc = np.asarray(y_yc, dtype=np.float64)
    n, N = y_yc.shape
    idx = np.arange(N) if cells is None else np.asarray(cells)
    M = len(idx)
    y = np.ascontiguousarray(y_yc[:, idx])
    fe = None if fext_yc is None else np.ascontiguousarray(np.asarray(fext_yc, dtype=np.float64)[:, idx])
    rh = None if rho is None else np.ascontiguousarray(np.asarray(rho, dtype=np.float64)[idx])
    proto = model.problem(1.0, None)
    o = make_opts(n, rtol, atol, ls=model.default_ls if ls is None else ls, group=group, **kw)
    st = (Stats * max(M, 1))()
    L = lib()
    nxt = [0]
    lk = threading.Lock()

    def worker():
        while True:
            with lk:
                c0 = nxt[0]
                nxt[0] = min(M, c0 + chunk)
            if c0 >= M:
                return
            c1 = min(M, c0 + chunk)
            sub = C.cast(C.byref(st, c0 * C.sizeof(Stats)), C.POINTER(Stats))
            L.orc_integrate_batch(C.byref(proto), C.byref(o), float(t0), float(tf), M, c0, c1, _dp(y),
                                  _dp(fe) if fe is not None else None, _dp(rh) if rh is not None else None, sub)

    ths = [threading.Thread(target=worker) for _ in range(max(1, threads))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    stats = {f: np.array([getattr(st[i], f) for i in range(M)]) for f in STAT_FIELDS}
    return y, stats
