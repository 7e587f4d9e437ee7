"""Mechanism table (mechanisms/<name>.json) -> straight-line, thread-per-cell
RHS and analytic Jacobian (paper_2405_01713_b200/csrc/gen/tpc_<name>.cuh).

Build-time only.  The paper's chemistry Jacobians are "generated offline,
mechanism-specific"; here every constant of the mechanism
(Arrhenius parameters, NASA-7 coefficients, stoichiometry, third-body
efficiencies, Troe parameters) is folded into generated code, so one thread
evaluates one cell with no table loads and no index arithmetic, and a warp
evaluates 32 cells in lock step (the per-cell integrator of csrc/bdf_tpc.cuh).

Physics (the paper's 0-D reactor "assumed constant internal
energy"; split form P:196-201) -- the same as csrc/mech_model.cuh:
  C_k = rho Y_k / W_k;  k_f = exp(ln A + beta ln T - Ea/(R_c T));
  [M] = sum_k alpha_k C_k;  Lindemann / Troe falloff;
  1/K_c = prod_reac e^{-g/RT} / prod_prod e^{-g/RT} * (R T / p_atm)^{dnu};
  q = k_f (prod_reac C - prod_prod C / K_c)  (times [M] for third body);
  wdot_k = sum_r nu_rk q_r;  dY_k/dt = W_k wdot_k / rho;
  dT/dt = -sum_k u_k wdot_k / (rho cv),  u_k = (h_k/RT - 1) R T.

Emitted device functions (struct Tpc_<name>):
  rhs(y[N], rho, f[N]) -> 0, or 1 if T <= 0 (recoverable RHS failure)
      y, f: per-thread register arrays after inlining.
  jac<SS>(y, rho, J, sc, Srt) -> same status (element stride S = SS, or Srt if SS = 0)
      y: N doubles at y[k*S]; J: row-major N x N at J[(i*N+j)*S];
      sc: scratch (NSC doubles at sc[m*S]), here the LU area that the matrix
      setup overwrites right after.  S = the workspace slot stride.
      Column-wise: pass 1 stores per-reaction kf, kr, dq/dT (and dq/d[M]);
      pass 2 builds one column of dwdot/dC in registers per species and
      the temperature row from it (chain rule through u_k and cv).
"""
from __future__ import annotations

import json
import re
import math
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
REPO = os.path.dirname(PKG)
RC = 1.98720425864083
RU = 8.31446261815324e7
PATM = 1013250.0
LN10 = 2.302585092994045684


def lit(x):
    x = float(x)
    return repr(x) if math.isfinite(x) else ("1e308" if x > 0 else "-1e308")


class Pool:
    """Floating constants of the generated code.  Values exactly representable in fp32
    are emitted as literals (SASS encodes them as immediates); every other constant
    goes to a __constant__ table, so FP64 instructions take it as a constant-bank
    operand instead of materialising it with two uniform-register moves."""

    def __init__(self, name):
        self.name = name
        self.vals = []
        self.idx = {}

    def __call__(self, x):
        x = float(x)
        if not math.isfinite(x) or struct.unpack("f", struct.pack("f", x))[0] == x:
            return lit(x)
        key = struct.pack("d", x)
        if key not in self.idx:
            self.idx[key] = len(self.vals)
            self.vals.append(x)
        return f"kc_{self.name}[{self.idx[key]}]"

    def table(self):
        body = ",\n  ".join(repr(v) for v in self.vals) or "0.0"
        return f"__constant__ double kc_{self.name}[{max(1, len(self.vals))}] = {{\n  {body}}};\n"


d = lit   # rebound per mechanism in generate()


NASA_SELECT = os.environ.get("BDFB_NASA_SELECT", "0") == "1"   # branch (default; selects measured 5% slower in K_rhs)


def _nasa_sel(A, tab, tm, body):
    """Branch-free NASA-7 range choice: `body(k, coeff)` with coeff(i, f) -> the expression
    `(lo ? f(a_low[i]) : f(a_high[i]))` (lanes of one warp may straddle Tmid: no divergent double path)."""
    for k, s in enumerate(tab["species"]):
        al, ah = s["nasa"]["low"], s["nasa"]["high"]

        def coeff(i, f=lambda x: x, al=al, ah=ah):
            vl, vh = f(al[i]), f(ah[i])
            return d(vl) if vl == vh else f"(lo ? {d(vl)} : {d(vh)})"
        body(k, coeff)


def _nasa(A, tab, tm, body):
    """Emit `body(k, coeffs, indent)` for both NASA-7 ranges (all Tmid equal)."""
    A(f"  if (T < {d(tm)}) {{\n")
    for k, s in enumerate(tab["species"]):
        body(k, s["nasa"]["low"])
    A("  } else {\n")
    for k, s in enumerate(tab["species"]):
        body(k, s["nasa"]["high"])
    A("  }\n")


def _rate(x, lnT="lnT", invT="invT", low=False):
    p = x["low"] if low else x
    if not low and x["b"] == 0 and x["Ea"] == 0:
        return d(x["A"])
    return f"fexp({d(math.log(p['A']))} + {d(p['b'])} * {lnT} - {d(p['Ea'] / RC)} * {invT})"


def _prod(names):
    return " * ".join(names) if names else "1.0"


def generate(name, out_dir):
    global d
    d = Pool(name)
    tab = json.load(open(os.path.join(REPO, "mechanisms", name + ".json")))
    sp = [s["name"] for s in tab["species"]]
    idx = {s: i for i, s in enumerate(sp)}
    K = len(sp)
    N = K + 1
    W = [s["W"] for s in tab["species"]]
    rx = tab["reactions"]
    NR = len(rx)
    tmids = {s["nasa"]["Tmid"] for s in tab["species"]}
    assert len(tmids) == 1, "generator assumes one common Tmid"
    tm = tmids.pop()
    tb = [r for r, x in enumerate(rx) if x["type"] != "elementary"]
    NTB = len(tb)
    # scratch layout of jac(): kf[NR], kr[NR], dqdT[NR], dqdM[NTB], h[K], cvk[K]
    O_KF, O_KR, O_DT, O_DM = 0, NR, 2 * NR, 3 * NR
    O_H = 3 * NR + NTB
    O_CV = O_H + K
    NSC = O_CV + K
    assert NSC <= N * N, "jac scratch must fit in the LU area"
    nu = []
    for x in rx:
        v = {}
        for s in x["reactants"]:
            v[idx[s]] = v.get(idx[s], 0) - 1
        for s in x["products"]:
            v[idx[s]] = v.get(idx[s], 0) + 1
        nu.append({k: c for k, c in v.items() if c != 0})

    L = []
    A = L.append
    A(f"// GENERATED by codegen/gen_tpc.py from mechanisms/{name}.json -- do not edit.\n")
    A(f"// {tab.get('provenance', '')}\n#pragma once\n#include \"../fexp.cuh\"\nnamespace bdfb {{\n")
    A("@@TABLE@@")
    A(f"struct Tpc_{name} {{\n")
    A(f"  static constexpr int K = {K}, N = {N}, NR = {NR}, NTB = {NTB}, NSC = {NSC};\n")
    A(f"  static constexpr const char* NAME = \"{name}\";\n")

    def thermo_common(A):
        A(f"  const double T = y{K};\n  if (!(T > 0.0)) return 1;\n")
        A("  const double lnT = log(T), invT = 1.0 / T, T2 = T * T, T3 = T2 * T, T4 = T3 * T;\n")
        A(f"  const bool lo = T < {d(tm)};   // NASA-7 range (selects, _nasa_sel)\n")
        A(f"  const double cRT = T * {d(RU / PATM)}, icRT = {d(PATM / RU)} * invT;\n")
        for k in range(K):
            A(f"  const double C{k} = rho * y{k} * {d(1.0 / W[k])};\n")
        for k in range(K):
            A(f"  double eg{k};\n")

    recip = sorted({idx[s] for x in rx if x["reversible"] for s in x["products"]})

    def post_thermo(A):
        for k in recip:
            A(f"  const double ieg{k} = 1.0 / eg{k};\n")
        if tb:
            A(f"  const double ctot = {' + '.join(f'C{k}' for k in range(K))};\n")

    def eg_body(k, a):
        # -g/RT = -(h/RT - s/R) = a0 (lnT - 1) + a1 T/2 + a2 T^2/6 + a3 T^3/12 + a4 T^4/20 - a5/T + a6
        A(f"    eg{k} = fexp({d(a[0])} * (lnT - 1.0) + {d(a[1] / 2)} * T + {d(a[2] / 6)} * T2 + {d(a[3] / 12)} * T3 + "
          f"{d(a[4] / 20)} * T4 - {d(a[5])} * invT + {d(a[6])});\n")

    def eg_body_sel(k, c):
        A(f"    eg{k} = fexp({c(0)} * (lnT - 1.0) + {c(1, lambda x: x / 2)} * T + {c(2, lambda x: x / 6)} * T2 + "
          f"{c(3, lambda x: x / 12)} * T3 + {c(4, lambda x: x / 20)} * T4 - {c(5)} * invT + {c(6)});\n")

    def reaction(A, r, x, deriv):
        """Emit the rate of progress q of reaction r (and its derivative data if deriv)."""
        reac = [idx[s] for s in x["reactants"]]
        prod = [idx[s] for s in x["products"]]
        typ = x["type"]
        dn = len(prod) - len(reac)
        A(f"  {{ // R{r}: {x['equation']}\n")
        A(f"    const double kinf = {_rate(x)};\n")
        const = x["b"] == 0 and x["Ea"] == 0
        A(f"    const double Cf = {_prod([f'C{i}' for i in reac])}, Cr = {_prod([f'C{i}' for i in prod])};\n")
        fac = {0: "", 1: " * cRT", -1: " * icRT", 2: " * (cRT * cRT)", -2: " * (icRT * icRT)"}[dn]
        if x["reversible"]:
            # 1/K_c = prod_reac e^{-g/RT} * prod_prod e^{+g/RT} (reciprocals once per species, no division here)
            A(f"    const double invKc = ({_prod([f'eg{i}' for i in reac])}) * ({_prod([f'ieg{i}' for i in prod])}){fac};\n")
        else:
            A("    const double invKc = 0.0;\n")
        A("    const double net = Cf - Cr * invKc;\n")
        if deriv:
            A(f"    const double dlnkinf = {'0.0' if const else f'({d(x['b'])} + {d(x['Ea'] / RC)} * invT) * invT'};\n")
            if x["reversible"]:
                hs = " + ".join([f"sc[{O_H + i}*S]" for i in prod]) + " - " + " - ".join([f"sc[{O_H + i}*S]" for i in reac])
                A(f"    const double dlnKc = ({hs} - {d(dn)}) * invT;\n")
            else:
                A("    const double dlnKc = 0.0;\n")
        if typ != "elementary":
            # [M] = sum_k alpha_k C_k = ctot + sum_{alpha_k != 1} (alpha_k - 1) C_k
            eff = x["efficiencies"]
            m = "ctot"
            for s in sp:
                e = eff.get(s, 1.0)
                if e != 1.0:
                    m = f"fma({d(e - 1.0)}, C{idx[s]}, {m})"
            A(f"    const double M = {m};\n")
        if typ in ("elementary", "three_body"):
            Mf = "M * " if typ == "three_body" else ""
            A(f"    const double kf = {Mf}kinf;\n")
            if deriv:
                A(f"    const double dkdT = kinf * dlnkinf;\n")
                if typ == "three_body":
                    A(f"    sc[{O_DM + tb.index(r)}*S] = kinf * net;\n")
                A(f"    sc[{O_DT + r}*S] = {'M * ' if typ == 'three_body' else ''}(dkdT * net + kinf * Cr * invKc * dlnKc);\n")
        else:
            lo = x["low"]
            A(f"    const double k0 = {_rate(x, low=True)};\n")
            A("    const double Pr = k0 * M / kinf;\n")
            A("    const double Pr1 = 1.0 / (1.0 + Pr);\n")
            if typ == "troe":
                t = x["troe"]
                A(f"    const double e3 = fexp(-T * {d(1.0 / t[1])}), e1 = fexp(-T * {d(1.0 / t[2])});\n")
                fc = f"{d(1 - t[0])} * e3 + {d(t[0])} * e1"
                if len(t) == 4:
                    A(f"    const double e2 = fexp({d(-t[3])} * invT);\n")
                    fc += " + e2"
                A(f"    const double Fc = {fc};\n")
                A("    const double lFc = log10(Fc);\n")
                A(f"    const double cc = {d(-0.4)} - {d(0.67)} * lFc, nn = 0.75 - {d(1.27)} * lFc;\n")
                A("    const double xx = log10(Pr) + cc;\n")
                A(f"    const double den = 1.0 / (nn - {d(0.14)} * xx);\n")
                A("    const double f1 = xx * den;\n")
                A("    const double q1 = 1.0 / (1.0 + f1 * f1);\n")
                A(f"    const double F = fexp(lFc * q1 * {d(LN10)});\n")
                if deriv:
                    dfc = f"-({d((1 - t[0]) / t[1])}) * e3 - ({d(t[0] / t[2])}) * e1"
                    if len(t) == 4:
                        dfc += f" + ({d(t[3])}) * invT * invT * e2"
                    A(f"    const double dFc = {dfc};\n")
                    A("    const double dlFdlPr = -lFc * 2.0 * f1 * (nn * den * den) * q1 * q1;\n")
                    A(f"    const double df1dlFc = ({d(-0.67)} * (nn - {d(0.14)} * xx) - xx * {d(-1.27 + 0.14 * 0.67)}) * den * den;\n")
                    A("    const double dlFdlFc = q1 - lFc * 2.0 * f1 * df1dlFc * q1 * q1;\n")
                    A(f"    const double dFdT = F * {d(LN10)} * dlFdlFc * (dFc / (Fc * {d(LN10)}));\n")
            else:
                A("    const double F = 1.0;\n")
                if deriv:
                    A("    const double dlFdlPr = 0.0, dFdT = 0.0;\n")
            A("    const double k = kinf * (Pr * Pr1 * F);\n")
            A("    const double kf = k;\n")
            if deriv:
                A("    const double dgdPr = F * Pr1 * Pr1 + Pr1 * F * dlFdlPr;\n")
                A(f"    const double dlnk0 = ({d(lo['b'])} + {d(lo['Ea'] / RC)} * invT) * invT;\n")
                A("    const double dkdT = k * dlnkinf + kinf * dgdPr * Pr * (dlnk0 - dlnkinf) + kinf * Pr * Pr1 * dFdT;\n")
                A(f"    sc[{O_DM + tb.index(r)}*S] = k0 * dgdPr * net;\n")
                A(f"    sc[{O_DT + r}*S] = dkdT * net + k * Cr * invKc * dlnKc;\n")
        A("    const double q = kf * net;\n")
        if deriv:
            A(f"    sc[{O_KF + r}*S] = kf;\n    sc[{O_KR + r}*S] = kf * invKc;\n")
        for i, v in sorted(nu[r].items()):
            if v == 1:
                A(f"    w{i} += q;\n")
            elif v == -1:
                A(f"    w{i} -= q;\n")
            else:
                A(f"    w{i} = fma({d(v)}, q, w{i});\n")
        A("  }\n")

    # ------------------------------------------------------------------ rhs
    rhs_start = len(L)
    A(f"  __device__ __forceinline__ static int rhs(const double (&yv)[{N}], double rho, double (&f)[{N}]) {{\n")
    for k in range(N):
        A(f"  const double y{k} = yv[{k}];\n")
    thermo_common(A)
    if NASA_SELECT:
        _nasa_sel(A, tab, tm, eg_body_sel)
    else:
        _nasa(A, tab, tm, eg_body)
    post_thermo(A)
    # cv = sum_k y_k cv_k before the reactions (same terms, same order as a fused tail): the y_k die here
    # instead of staying live across the reaction loop
    A("  double cv = 0.0;\n")

    def cv_body(k, a):
        A(f"    cv = fma(y{k} * {d(RU / W[k])}, {d(a[0] - 1)} + T * ({d(a[1])} + T * ({d(a[2])} + T * ({d(a[3])} + T * {d(a[4])}))), cv);\n")

    def cv_body_sel(k, c):
        A(f"    cv = fma(y{k} * {d(RU / W[k])}, {c(0, lambda x: x - 1)} + T * ({c(1)} + T * ({c(2)} + T * ({c(3)} + T * {c(4)}))), cv);\n")
    if NASA_SELECT:
        _nasa_sel(A, tab, tm, cv_body_sel)
    else:
        _nasa(A, tab, tm, cv_body)
    for k in range(K):
        A(f"  double w{k} = 0.0;\n")
    for r, x in enumerate(rx):
        reaction(A, r, x, False)
    A("  double su = 0.0;\n")

    def tail_body(k, a):
        A(f"    su = fma({d(a[0] - 1)} + T * ({d(a[1] / 2)} + T * ({d(a[2] / 3)} + T * ({d(a[3] / 4)} + T * {d(a[4] / 5)}))) + "
          f"{d(a[5])} * invT, w{k}, su);\n")
    def tail_body_sel(k, c):
        A(f"    su = fma({c(0, lambda x: x - 1)} + T * ({c(1, lambda x: x / 2)} + T * ({c(2, lambda x: x / 3)} + T * ({c(3, lambda x: x / 4)} + T * {c(4, lambda x: x / 5)}))) + "
          f"{c(5)} * invT, w{k}, su);\n")
    if NASA_SELECT:
        _nasa_sel(A, tab, tm, tail_body_sel)
    else:
        _nasa(A, tab, tm, tail_body)
    A("  const double irho = 1.0 / rho;\n")
    for k in range(K):
        A(f"  f[{k}] = {d(W[k])} * w{k} * irho;\n")
    A(f"  f[{K}] = -su * {d(RU)} * T / (rho * cv);\n  return 0;\n  }}\n\n")
    # rhs_sm<SS>: the same operations with e^{-g/RT} and its reciprocal in a per-thread shared-memory column
    # (sm[k SS] and sm[(K + k) SS], SS = the block's thread count) instead of registers: 2K fewer live values
    # across the reaction loop (the register-resident version spills at 168 registers)
    src = "".join(L[rhs_start:])
    src = src.replace(f"static int rhs(const double (&yv)[{N}], double rho, double (&f)[{N}]) {{",
                      f"static int rhs_sm(const double (&yv)[{N}], double rho, double (&f)[{N}], "
                      f"double* __restrict__ sm) {{", 1)
    src = src.replace("  __device__ __forceinline__ static int rhs_sm", "  template <int SS>\n  __device__ __forceinline__ static int rhs_sm", 1)
    src = re.sub(r"  double eg(\d+);\n", "", src)
    src = re.sub(r"const double ieg(\d+) = 1\.0 / eg(\d+);",
                 lambda m: f"sm[{K + int(m.group(1))} * SS] = 1.0 / sm[{int(m.group(2))} * SS];", src)
    src = re.sub(r"(?<![A-Za-z0-9_])ieg(\d+)\b", lambda m: f"sm[{K + int(m.group(1))} * SS]", src)
    src = re.sub(r"(?<![A-Za-z0-9_])eg(\d+)\b", lambda m: f"sm[{int(m.group(1))} * SS]", src)
    # reads through a volatile view, so that the compiler reloads them from shared memory instead of keeping
    # the stored values live in registers (which would undo the point of the variant)
    src = src.replace("sm[", "sv[")
    src = re.sub(r"^(\s*)sv\[([^\]]*)\] = ", lambda m: f"{m.group(1)}sm[{m.group(2)}] = ", src, flags=re.M)
    src = src.replace("double* __restrict__ sm) {\n", "double* __restrict__ sm) {\n  volatile const double* sv = sm;\n", 1)
    A(src)

    # ------------------------------------------------------------------ jac
    jac_start = len(L)
    A("  template <long long SS>  // compile-time element stride (0: runtime Srt)\n")
    A("  __device__ __noinline__ static int jac(const double* __restrict__ yp, double rho, double* __restrict__ J, "
      "double* __restrict__ sc, long long Srt) {\n")
    A("  const long long S = SS ? SS : Srt;\n")
    for k in range(N):
        A(f"  const double y{k} = yp[{k}*S];\n")
    thermo_common(A)

    def jac_thermo(k, a):
        eg_body(k, a)
        # h/RT into scratch (for dlnKc), cv_k = (cp_k/R - 1) R / W_k, u_k/W_k, dcp_k/dT
        A(f"    sc[{O_H + k}*S] = {d(a[0])} + T * ({d(a[1] / 2)} + T * ({d(a[2] / 3)} + T * ({d(a[3] / 4)} + T * {d(a[4] / 5)}))) + {d(a[5])} * invT;\n")
        A(f"    sc[{O_CV + k}*S] = ({d(a[0] - 1)} + T * ({d(a[1])} + T * ({d(a[2])} + T * ({d(a[3])} + T * {d(a[4])})))) * {d(RU / W[k])};\n")
    _nasa(A, tab, tm, jac_thermo)
    post_thermo(A)
    for k in range(K):
        A(f"  double w{k} = 0.0;\n")
    for r, x in enumerate(rx):
        reaction(A, r, x, True)
    # cv, su, scw, dcv; uoW_k (registers for pass 2)
    A("  double cv = 0.0, su = 0.0, scw = 0.0, dcv = 0.0;\n")
    for k in range(K):
        A(f"  double uoW{k};\n")

    def jac_tail(k, a):
        A(f"    {{ const double hk = sc[{O_H + k}*S], cvk = sc[{O_CV + k}*S];\n")
        A(f"      uoW{k} = (hk - 1.0) * {d(RU)} * T * {d(1.0 / W[k])};\n")
        A(f"      cv = fma(y{k}, cvk, cv);\n")
        A(f"      su = fma(uoW{k} * {d(W[k])}, w{k}, su);\n")
        A(f"      scw = fma(cvk * {d(W[k])}, w{k}, scw);\n")
        A(f"      dcv = fma(y{k} * {d(RU / W[k])}, {d(a[1])} + T * ({d(2 * a[2])} + T * ({d(3 * a[3])} + T * {d(4 * a[4])})), dcv); }}\n")
    _nasa(A, tab, tm, jac_tail)
    A("  const double icv = 1.0 / cv, irho = 1.0 / rho;\n")
    A("  const double fT0 = -su * irho * icv;\n")
    p1_end = len(L)
    col_start = []
    # pass 2: species columns
    for j in range(K):
        col_start.append(len(L))
        A(f"  {{ // column {j} ({sp[j]})\n")
        rows = {}
        terms = []
        for r, x in enumerate(rx):
            reac = [idx[s] for s in x["reactants"]]
            prod = [idx[s] for s in x["products"]]
            parts = []
            for o in range(len(reac)):
                if reac[o] == j:
                    others = reac[:o] + reac[o + 1:]
                    parts.append(" * ".join([f"sc[{O_KF + r}*S]"] + [f"C{i}" for i in others]))
            pparts = []
            if x["reversible"]:
                for o in range(len(prod)):
                    if prod[o] == j:
                        others = prod[:o] + prod[o + 1:]
                        pparts.append(" * ".join([f"sc[{O_KR + r}*S]"] + [f"C{i}" for i in others]))
            tbterm = None
            if x["type"] != "elementary":
                e = x["efficiencies"].get(sp[j], 1.0)
                if e != 0.0:
                    tbterm = f"sc[{O_DM + tb.index(r)}*S]" + ("" if e == 1.0 else f" * {d(e)}")
            if not parts and not pparts and tbterm is None:
                continue
            if not nu[r]:
                continue
            expr = " + ".join(parts) if parts else "0.0"
            for pp in pparts:
                expr += f" - {pp}"
            if tbterm:
                expr += f" + {tbterm}"
            terms.append((r, expr))
            for i in nu[r]:
                rows[i] = True
        for i in sorted(rows):
            A(f"    double c{i} = 0.0;\n")
        for r, expr in terms:
            A(f"    {{ const double dq = {expr};\n")
            for i, v in sorted(nu[r].items()):
                if v == 1:
                    A(f"      c{i} += dq;\n")
                elif v == -1:
                    A(f"      c{i} -= dq;\n")
                else:
                    A(f"      c{i} = fma({d(v)}, dq, c{i});\n")
            A("    }\n")
        A("    double s = 0.0;\n")
        for i in range(K):
            if i in rows:
                A(f"    {{ const double v = c{i} * {d(W[i] / W[j])}; J[{i * N + j}*S] = v; s = fma(uoW{i}, v, s); }}\n")
            else:
                A(f"    J[{i * N + j}*S] = 0.0;\n")
        A(f"    J[{K * N + j}*S] = -s * icv - fT0 * sc[{O_CV + j}*S] * icv;\n")
        A("  }\n")
    # temperature column
    col_start.append(len(L))
    A("  {\n")
    rowsT = {}
    for r in range(NR):
        for i in nu[r]:
            rowsT.setdefault(i, []).append(r)
    A("    double s = 0.0;\n")
    for i in range(K):
        if i in rowsT:
            A("    { double c = 0.0;\n")
            for r in rowsT[i]:
                v = nu[r][i]
                if v == 1:
                    A(f"      c += sc[{O_DT + r}*S];\n")
                elif v == -1:
                    A(f"      c -= sc[{O_DT + r}*S];\n")
                else:
                    A(f"      c = fma({d(v)}, sc[{O_DT + r}*S], c);\n")
            A(f"      const double v = {d(W[i])} * c * irho; J[{i * N + K}*S] = v; s = fma(uoW{i}, v, s); }}\n")
        else:
            A(f"    J[{i * N + K}*S] = 0.0;\n")
    A(f"    J[{K * N + K}*S] = -scw * irho * icv - s * icv - fT0 * dcv * icv;\n")
    A("  }\n")
    col_end = len(L)
    A("  return 0;\n  }\n")
    # jac_cm: the same body with y at yp[k * SY] (e.g. a warp-blocked SoA state), J column-major and
    # contiguous (J(i, j) at J[j * N + i], the split kernel's per-cell record) and contiguous scratch
    body = "".join(L[jac_start:])
    body = body.replace("  template <long long SS>  // compile-time element stride (0: runtime Srt)\n",
                        "  template <long long SY>  // element stride of y; J column-major, contiguous\n")
    body = body.replace("static int jac(const double* __restrict__ yp, double rho, double* __restrict__ J, "
                        "double* __restrict__ sc, long long Srt) {\n",
                        "static int jac_cm(const double* __restrict__ yp, double rho, double* __restrict__ J, "
                        "double* __restrict__ sc) {\n")
    body = body.replace("  const long long S = SS ? SS : Srt;\n", "")
    body = re.sub(r"yp\[(\d+)\*S\]", lambda m: f"yp[{m.group(1)}*SY]", body)
    body = re.sub(r"J\[(\d+)\*S\]", lambda m: f"J[{(int(m.group(1)) % N) * N + int(m.group(1)) // N}]", body)
    body = re.sub(r"sc\[(\d+)\*S\]", lambda m: f"sc[{m.group(1)}]", body)
    assert "*S]" not in body, "unconverted stride in jac_cm"
    A(body)
    # jac_p1 / jac_col: jac_cm split in two passes with the same operations (so the same J bit for bit).
    # Pass 1 (one thread per cell): thermo, every reaction's kf, kr, dq/dT, dq/d[M], the energy sums, then
    # C_k, u_k/W_k and the scalars into the scratch sc.  Pass 2 (one thread per (cell, column j), warp-uniform
    # j): column j of J from the scratch.  The Jacobian list of one SPLIT iteration is ~10^4 cells, so a
    # thread per cell leaves most of the GPU idle behind one long serial chain; the column pass has N times
    # the threads.  Scratch offsets after jac's: C_k at O_C, u_k/W_k at O_U, then icv, irho, fT0, scw, dcv.
    O_C = NSC
    O_U = O_C + K
    O_SC = O_U + K
    NSC2 = O_SC + 5

    def conv(t):
        t = re.sub(r"yp\[(\d+)\*S\]", lambda m: f"yp[{m.group(1)}*SY]", t)
        t = re.sub(r"J\[(\d+)\*S\]", lambda m: f"J[{(int(m.group(1)) % N) * N + int(m.group(1)) // N}]", t)
        t = re.sub(r"sc\[(\d+)\*S\]", lambda m: f"sc[{m.group(1)}]", t)
        return t
    p1 = "".join(L[jac_start:p1_end])
    p1 = p1.replace("  template <long long SS>  // compile-time element stride (0: runtime Srt)\n",
                    "  template <long long SY, long long SC>  // element strides of y and of the scratch\n")
    p1 = p1.replace("__device__ __noinline__ static int jac(const double* __restrict__ yp, double rho, "
                    "double* __restrict__ J, double* __restrict__ sc, long long Srt) {\n",
                    "__device__ __forceinline__ static int jac_p1(const double* __restrict__ yp, double rho, "
                    "double* __restrict__ sc) {\n")
    p1 = p1.replace("  const long long S = SS ? SS : Srt;\n", "")
    p1 = conv(p1)
    for k in range(K):
        p1 += f"  sc[{O_C + k}] = C{k};\n  sc[{O_U + k}] = uoW{k};\n"
    p1 += (f"  sc[{O_SC}] = icv;\n  sc[{O_SC + 1}] = irho;\n  sc[{O_SC + 2}] = fT0;\n  sc[{O_SC + 3}] = scw;\n"
           f"  sc[{O_SC + 4}] = dcv;\n  return 0;\n  }}\n\n")
    p1 = re.sub(r"sc\[(\d+)\]", lambda m: f"sc[{m.group(1)}*SC]", p1)
    assert "*S]" not in p1, "unconverted stride in jac_p1"
    A(p1)
    # ---- parted pass 1 (jac_part<SY, SC>(P, ...) + jac_sum<SY, SC>): the reactions dealt round-robin to NPART
    # parts (one warp-uniform part per thread), so a Jacobian list of ~10^4 cells runs NPART x the threads over
    # NPART x shorter chains.  Part P evaluates the thermo of the species its reversible reactions need (h/RT
    # into the scratch: identical values from every part), its reactions' kf, kr, dq/dT, dq/d[M] (the
    # expressions of jac) and its partial production rates.  jac_sum (one thread per cell, after the parts):
    # C_k, cv_k, u_k/W_k, cv, dcv (jac_tail's expressions), the production rates added in part order, su, scw,
    # icv, irho, fT0 (the rates are summed in another order than jac's: J agrees with it to rounding, R19).
    # Scratch: jac's layout, then WP[P][k] at O_WP + P K + k.
    NPART = 4
    O_WP = NSC2
    NSC3 = O_WP + NPART * K
    A(f"  static constexpr int NPART = {NPART}, NSC3 = {NSC3};   // parts of jac_part; its scratch doubles\n")
    touched_all = []
    for P in range(NPART):
        rs = [r for r in range(NR) if r % NPART == P]
        need = set()
        for r in rs:
            x = rx[r]
            if x["reversible"]:
                need |= {idx[t] for t in x["reactants"]} | {idx[t] for t in x["products"]}
        touched = sorted({i for r in rs for i in nu[r]})
        touched_all.append(touched)
        B = []
        AB = B.append
        AB(f"  template <long long SY, long long SC>\n  __device__ __forceinline__ static int jac_part{P}("
           f"const double* __restrict__ yp, double rho, double* __restrict__ sc) {{\n")
        for k in range(N):
            AB(f"  const double y{k} = yp[{k}*SY];\n")
        thermo_common(AB)

        def th(k, a, AB=AB, need=need):
            if k not in need:
                return
            AB(f"    eg{k} = fexp({d(a[0])} * (lnT - 1.0) + {d(a[1] / 2)} * T + {d(a[2] / 6)} * T2 + {d(a[3] / 12)} * T3 + "
               f"{d(a[4] / 20)} * T4 - {d(a[5])} * invT + {d(a[6])});\n")
            AB(f"    sc[{O_H + k}*S] = {d(a[0])} + T * ({d(a[1] / 2)} + T * ({d(a[2] / 3)} + T * ({d(a[3] / 4)} + T * {d(a[4] / 5)}))) + {d(a[5])} * invT;\n")
        if need:
            _nasa(AB, tab, tm, th)
        for k in recip:
            if k in need:
                AB(f"  const double ieg{k} = 1.0 / eg{k};\n")
        if tb:
            AB(f"  const double ctot = {' + '.join(f'C{k}' for k in range(K))};\n")
        for k in touched:
            AB(f"  double w{k} = 0.0;\n")
        for r in rs:
            reaction(AB, r, rx[r], True)
        for k in touched:
            AB(f"  sc[{O_WP + P * K + k}*S] = w{k};\n")
        AB("  return 0;\n  }\n")
        body = "".join(B)
        body = re.sub(r"  double eg(\d+);\n", lambda m: m.group(0) if int(m.group(1)) in need else "", body)
        body = re.sub(r"sc\[(\d+)\*S\]", lambda m: f"sc[{m.group(1)}*SC]", body)
        assert "*S]" not in body, "unconverted stride in jac_part"
        A(body)
    A("  template <long long SY, long long SC>\n  __device__ __forceinline__ static int jac_part(int P, "
      "const double* __restrict__ yp, double rho, double* __restrict__ sc) {\n  switch (P) {\n")
    for P in range(NPART):
        A(f"  case {P}: return jac_part{P}<SY, SC>(yp, rho, sc);\n")
    A("  }\n  return 0;\n  }\n")
    B = []
    AB = B.append
    AB("  template <long long SY, long long SC>\n  __device__ __forceinline__ static int jac_sum("
       "const double* __restrict__ yp, double rho, double* __restrict__ sc) {\n")
    for k in range(N):
        AB(f"  const double y{k} = yp[{k}*SY];\n")
    AB(f"  const double T = y{K};\n  if (!(T > 0.0)) return 1;\n  const double invT = 1.0 / T;\n")
    for k in range(K):
        AB(f"  sc[{O_C + k}*S] = rho * y{k} * {d(1.0 / W[k])};\n")
    AB("  double cv = 0.0, su = 0.0, scw = 0.0, dcv = 0.0;\n")

    def tails(k, a, AB=AB):
        parts_k = [P for P in range(NPART) if k in touched_all[P]]
        wsum = " + ".join(f"sc[{O_WP + P * K + k}*S]" for P in parts_k) if parts_k else "0.0"
        AB(f"    {{ const double hk = {d(a[0])} + T * ({d(a[1] / 2)} + T * ({d(a[2] / 3)} + T * ({d(a[3] / 4)} + T * {d(a[4] / 5)}))) + {d(a[5])} * invT;\n")
        AB(f"      const double cvk = ({d(a[0] - 1)} + T * ({d(a[1])} + T * ({d(a[2])} + T * ({d(a[3])} + T * {d(a[4])})))) * {d(RU / W[k])};\n")
        AB(f"      sc[{O_CV + k}*S] = cvk;\n")
        AB(f"      const double uoW = (hk - 1.0) * {d(RU)} * T * {d(1.0 / W[k])};\n")
        AB(f"      sc[{O_U + k}*S] = uoW;\n")
        AB(f"      const double w = {wsum};\n")
        AB(f"      cv = fma(y{k}, cvk, cv);\n")
        AB(f"      su = fma(uoW * {d(W[k])}, w, su);\n")
        AB(f"      scw = fma(cvk * {d(W[k])}, w, scw);\n")
        AB(f"      dcv = fma(y{k} * {d(RU / W[k])}, {d(a[1])} + T * ({d(2 * a[2])} + T * ({d(3 * a[3])} + T * {d(4 * a[4])})), dcv); }}\n")
    _nasa(AB, tab, tm, tails)
    AB("  const double icv = 1.0 / cv, irho = 1.0 / rho;\n")
    AB(f"  sc[{O_SC}*S] = icv;\n  sc[{O_SC + 1}*S] = irho;\n  sc[{O_SC + 2}*S] = -su * irho * icv;\n"
       f"  sc[{O_SC + 3}*S] = scw;\n  sc[{O_SC + 4}*S] = dcv;\n  return 0;\n  }}\n")
    body = "".join(B)
    body = re.sub(r"sc\[(\d+)\*S\]", lambda m: f"sc[{m.group(1)}*SC]", body)
    assert "*S]" not in body, "unconverted stride in jac_sum"
    A(body)
    A(f"  static constexpr int NSC2 = {NSC2};   // scratch doubles of jac_p1 / jac_col\n")
    A("  // column j (0..N-1) of the column-major J from jac_p1's scratch (element stride SC)\n")
    A("  template <long long SC>\n  __device__ __forceinline__ static void jac_col(int j, const double* __restrict__ sc, "
      "double* __restrict__ J) {\n")
    A(f"  const double icv = sc[{O_SC}*SC], irho = sc[{O_SC + 1}*SC], fT0 = sc[{O_SC + 2}*SC], "
      f"scw = sc[{O_SC + 3}*SC], dcv = sc[{O_SC + 4}*SC];\n")
    A("  (void)irho; (void)scw; (void)dcv; (void)fT0;\n  switch (j) {\n")
    for c in range(N):
        seg = "".join(L[col_start[c]:(col_start[c + 1] if c + 1 < N else col_end)])
        seg = conv(seg)
        seg = re.sub(r"(?<![A-Za-z0-9_])C(\d+)\b", lambda m: f"sc[{O_C + int(m.group(1))}]", seg)
        seg = re.sub(r"(?<![A-Za-z0-9_])uoW(\d+)\b", lambda m: f"sc[{O_U + int(m.group(1))}]", seg)
        seg = re.sub(r"sc\[(\d+)\]", lambda m: f"sc[{m.group(1)}*SC]", seg)
        assert "*S]" not in seg, "unconverted stride in jac_col"
        A(f"  case {c}:\n{seg}  break;\n")
    A("  }\n  }\n")
    A("};\n}  // namespace bdfb\n")
    os.makedirs(out_dir, exist_ok=True)
    p = os.path.join(out_dir, f"tpc_{name}.cuh")
    src = "".join(L).replace("@@TABLE@@", d.table())
    if not os.path.exists(p) or open(p).read() != src:
        open(p, "w").write(src)
    return p


MECHANISMS = ["h2_lidryer", "drm19_class", "gri53_class"]   # gri53: its RHS only is used (C5)


def main(argv=None):
    out = os.path.join(PKG, "csrc", "gen")
    for m in (argv or MECHANISMS):
        print(generate(m, out))


if __name__ == "__main__":
    main(sys.argv[1:])
