"""Benchmark: cell ODE integrations per second per outer step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A "step" is one outer fluid step of the hot path: bdfb_integrate of every cell
of the workload from t0 to t0 + dt_CFD (per-cell BDF: RHS, Jacobian, Newton,
LU, WRMS, step/order control -- SURVEY.md §8(a)), restarted each step from the
same pristine synthetic field (copied in untimed; the state alone is 2.9 GB,
far larger than the 126 MB L2).  Multi-GPU (torchrun): by default the config's
fixed grid is dealt over the ranks in block-cyclic 16^3 tiles (strong scaling,
BASELINE "256^3 cells sharded over 2/4/8 B200"; --scaling weak gives every rank
a full grid); no collective on the data path; the timed duration is the max
over ranks and value = all ranks' cells / that time.

The JSON line carries the device-timed value, the FP64 roofline of the
integrator kernel, the CPU oracle timed on the host cores (cpu_baseline), an
end-to-end number through the host-buffer C-ABI call (e2e), the GPU clocks
sampled during the timed region and the per-cell statistics behind the flop
count.  `--impl reference` times the CPU oracle instead (the reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    # id: (model, mech table, n, L, dt_CFD, rtol, atol, description)
    "C1": ("robertson", None, 3, None, 40.0, 1e-4, (1e-8, 1e-14, 1e-6),
           "C1 Robertson 3-species kinetics, 1024 cells, t in [0,40], rtol 1e-4"),
    "C2": ("nyx_kwh", None, 1, 128, 3.0e15, 1e-6, 1e-10,
           "C2 Nyx-style scalar heating/cooling (KWH96 form, CVDiag), 128^3 cells, dt 3e15 s"),
    "C3": ("h2", "h2_lidryer", 10, 64, 1e-5, 1e-6, 1e-10,
           "C3 H2/air (9 species + T, n=10) flame field on 64^3 cells, dt_CFD 1e-5 s"),
    "C4": ("drm19", "drm19_class", 22, 256, 1e-5, 1e-6, 1e-10,
           "C4 DRM19-class CH4/air (21 species + T, n=22) flame field on 256^3 cells, dt_CFD 1e-5 s"),
    # the paper's lockstep batch (row a12) on the DRM19-class mechanism at C5's per-GPU cell count
    # (256^3 / 8 GPUs = 128^3): the global-norm path of the generated thread-per-cell kernels.
    # BASELINE configs[4]: the ~53-species mechanism on 256^3 cells over 8 B200 in the global-norm mode; one GPU
    # runs its 1/8 share (a 256 x 256 x 32 slab = 128^3 cells); rank r of k <= 8 ranks its slab r (weak scaling)
    "C5": ("gri53", "gri53_class", 54, 256, 1e-6, 1e-6, 1e-10,
           "C5 GRI-3.0-class CH4/air (53 species + T, n=54, 325 reactions) flame field, global-norm mode (one "
           "lockstep batch, batch-wide WRMS), 256^3 grid in 8 z-slabs of 128^3 cells (one per GPU), dt_CFD 1e-6 s"),
    # C5's mechanism and grid share per cell (the north_star's per-cell mode) instead of the lockstep batch
    "C5P": ("gri53", "gri53_class", 54, 256, 1e-6, 1e-6, 1e-10,
            "C5P GRI-3.0-class CH4/air (53 species + T, n=54, 325 reactions) flame field, per-cell mode (SPLIT), "
            "256^3 grid in 8 z-slabs of 128^3 cells (one per GPU), dt_CFD 1e-6 s"),
    "G4": ("drm19", "drm19_class", 22, 128, 1e-5, 1e-6, 1e-10,
           "G4 global-norm mode (lockstep batch, batch-wide WRMS) on the DRM19-class flame field, 128^3 cells "
           "(C5's per-GPU share at 8 GPUs), dt_CFD 1e-5 s"),
}
GLOBAL_CFGS = {"G4", "C5"}
C5_SLAB = 256 ** 3 // 8            # cells per GPU in C5
METRIC = "cell ODE integrations/sec per outer step"
UNIT = "cells/s"
FP64_FMA_PER_SM_CLK = 64        # B200 FP64 units per SM (sm_100a): 148 x 64 x 2 x 1.965 GHz = 37.2 TF
SMS = 148
SM_MAX_MHZ = 1965.0
# FP64 flops charged per exp / log call ("weighted by its FP64-pipe instruction count, measured
# once on the box"): 2 DFMA + DADD + DMUL executed per call of the GPU's exp (fexp) and log, from ncu on
# exp/probe/transc_probe.cu (profiles/r2/transc_weights.json); fallback: the static SASS counts of the same probe.
TRANSC_STATIC = {"exp": 31, "log": 46, "source": "static SASS count of exp/probe/transc_probe.cu (cuobjdump)"}


def transc_weights():
    try:
        with open(os.path.join(REPO, "profiles", "r2", "transc_weights.json")) as f:
            w = json.load(f)
        # the logs of the definition are one ln T per RHS plus log10 (Troe); charged at the log10 cost
        return {"exp": float(w["fexp"]["flops_per_call"]), "log": float(w["log10"]["flops_per_call"]),
                "source": "ncu executed 2 DFMA + DADD + DMUL per call of fexp / log10 "
                          "(profiles/r2/transc_weights.json)"}
    except Exception:
        return dict(TRANSC_STATIC)


def _gen_counts(mech):
    hdr = open(os.path.join(REPO, "paper_2405_01713_b200", "csrc", "gen", f"mech_{mech}.cuh")).read()
    return lambda k: int(re.search(rf"{k} = (\d+)", hdr).group(1))  # noqa: E731


# ------------------------------------------------------------------ inputs
def rank_cells(cfg, rank=0, world=1, scaling="strong", cells_per_rank=None):
    """Global cell indices this rank integrates.  strong: the config's fixed grid shared by the ranks -- 16^3
    tiles dealt block-cyclically (parallel.block_cyclic_cells) for the per-cell grids, contiguous
    256-aligned slabs for the global-norm batch and C1's 1024 cells; weak: `cells_per_rank` (default the
    config's grid) per rank, rank r owning global cells r N .. (r+1) N - 1 of one larger seeded field."""
    from paper_2405_01713_b200 import parallel as PL
    L = CONFIGS[cfg][3]
    total = 1024 if cfg == "C1" else L ** 3
    if cfg in ("C5", "C5P") and not cells_per_rank:     # the 256^3 grid's z-slab r (of 8): fixed share per GPU
        if world > 8:
            raise SystemExit("C5 is defined on 8 GPUs (256^3 / 8 cells each)")
        return np.arange(rank * C5_SLAB, (rank + 1) * C5_SLAB), C5_SLAB * world
    if scaling == "weak" or cells_per_rank:
        N = cells_per_rank or total
        return np.arange(*PL.shard(rank, world, N)), N * world
    if world == 1:
        return np.arange(total), total
    if cfg == "C1" or cfg in GLOBAL_CFGS:
        return np.arange(*PL.contiguous_cells(rank, world, total, 1 if cfg == "C1" else 256)), total
    return PL.block_cyclic_cells(rank, world, L, 16), total


def make_inputs(cfg, rank=0, cells_per_rank=None, world=1, scaling="strong"):
    """This rank's cells of the seeded field (identical values under any partition: synth is counter-based)."""
    from synth import flame_field, nyx_field, robertson_field
    model, mech, n, L, dt, rtol, atol, _ = CONFIGS[cfg]
    cells, total = rank_cells(cfg, rank, world, scaling, cells_per_rank)
    if cfg == "C1":
        return robertson_field(total, cells=cells), None, None, np.arange(len(cells))
    if cfg == "C2":
        e, rho, fe = nyx_field(L, cells=cells, dt=dt)
        return e, rho, fe, None
    y, rho, F, prog = flame_field(mech, L, cells=cells, dt=dt)
    return y, rho, F, prog


def unit_flops(cfg):
    """Algorithmic FP64 flops per unit of work: one RHS, one Jacobian, one matrix setup
    (M = I - gamma J and the reciprocal-multiply LU), one Newton solve (+ its vector updates and norm),
    one attempt (predict, weights, coefficients, error test), one accepted step (completion, PREPARE_NEXT)."""
    model, mech, n, *_ = CONFIGS[cfg]
    w = transc_weights()
    if mech:
        g = _gen_counts(mech)
        f_rhs = g("FLOPS_RHS_ARITH") + w["exp"] * g("RHS_EXPS") + w["log"] * g("RHS_LOGS")
        f_jac = g("FLOPS_JAC_ARITH") + w["exp"] * g("JAC_EXPS") + w["log"] * g("JAC_LOGS")
    elif model == "robertson":
        f_rhs, f_jac = 12, 10
    else:  # nyx_kwh: ~12 regula-falsi evaluations x (~16 transcendental + 40 arith) + cooling sum
        f_rhs, f_jac = 12 * (16 * w["exp"] + 40) + 20 * w["exp"] + 60, 0
    # krylov: one GMRES iteration besides its RHS call (Jv quotient and scaling 6n, modified Gram-Schmidt against
    # ~2 basis vectors 8n, norm 2n, Givens ~20); erk_attempt: the stage combinations 14n, the solution 8n, the
    # error estimate 10n and its norm 3n of one ERK attempt
    return {"rhs": f_rhs, "jac": f_jac, "setup": (2 * (n - 1) * n * (2 * n - 1)) // 6 + n * (n - 1) // 2 + n + 2 * n * n,
            "solve": 2 * n * n - n + 9 * n, "attempt": 26 * n + 60, "step": 11 * n + 80, "krylov": 16 * n + 20,
            "erk_attempt": 35 * n + 20}


def phase_flops(cfg, st, method="bdf", ls="dense"):
    """Algorithmic FP64 flops of one integrate per SPLIT kernel phase (the whole step is their sum):
    K_rhs = nfe F_rhs, K_jac = nje F_jac, K_lu = nsetups F_setup, K_ctl = Newton solves + vector passes +
    control.  Global-norm mode: batch counters, every batch step does the work for every cell."""
    u = unit_flops(cfg)
    att = st["nst"] + st["netf"] + st["ncfn"]
    if method == "erk4":   # one kernel: RHS calls and the stage algebra; no algebraic solver
        return {"rhs": st["nfe"] * u["rhs"], "ctl": (st["nst"] + st["netf"]) * u["erk_attempt"], "jac": 0, "lu": 0}
    nli = st.get("nli", 0)   # GMRES: one RHS call per Krylov iteration (Jv quotient)
    ph = {"rhs": (st["nfe"] + nli) * u["rhs"], "jac": st["nje"] * u["jac"], "lu": st["nsetups"] * u["setup"],
          "ctl": st["nni"] * u["solve"] + att * u["attempt"] + st["nst"] * u["step"] + nli * u["krylov"]}
    if ls != "dense":      # matrix-free: no J, no LU; CVDiag's setup is one RHS call (in nfe) + 6n, its solve 2n
        n = CONFIGS[cfg][2]
        ph["jac"], ph["lu"] = 0, 0
        ph["ctl"] = st["nni"] * (2 * n + 9 * n) + st["nsetups"] * 6 * n + att * u["attempt"] + st["nst"] * u["step"] + \
            nli * u["krylov"]
    if cfg in GLOBAL_CFGS:
        ph = {k: v * st["n_cells"] for k, v in ph.items()}
    return ph


def flop_model(cfg, st, method="bdf"):
    """Algorithmic FP64 flops of one integrate (whole step) from the aggregate per-cell statistics."""
    return sum(phase_flops(cfg, st, method).values())


def hbm_bytes_global(cfg, st):
    """Algorithmic HBM bytes of one global-norm-mode integrate: per Newton solve the
    cell's LU (8 n^2) + pivots/1/U (16 n) + del, acor r/w, b (32 n); per RHS y, F in, f out (24 n + 8);
    per setup J r/w + LU w (24 n^2); per norm 16 n; per step the Nordsieck updates (2 (q+1) 8 n, q ~ 3)."""
    n = CONFIGS[cfg][2]
    per_cell = (st["nni"] * (8 * n * n + 16 * n + 32 * n) + st["nfe"] * (24 * n + 8) +
                st["nsetups"] * 24 * n * n + (st["nni"] + st["nst"]) * 16 * n + st["nst"] * 64 * n)
    return per_cell * st["n_cells"]


TS_RECORD_BYTES = 408          # struct TS record of the SPLIT slot pool (TS_STRIDE = 51 doubles, csrc/bdf_tpc.cuh)
QBAR = 3                       # mean BDF order assumed by the byte model (zn[0..q] rows moved per pass)


def ctl_bytes(cfg, st):
    """Bytes the SPLIT control kernel K_ctl must move per integrate: every visit of a slot
    (one per consumed RHS value and one per resumed setup) reads and writes the cell's TS record; a
    consumed Newton residual reads fr, zn[1], acor and writes del (32n + 4); a Newton solve streams the
    LU record (8n^2 + 12n) and moves del, acor (r/w), ewt, zn[0], yq (48n); an attempt reads and writes
    zn[0..q] once (the deferred step completion, order change, rescale and predictor fused: 16 (q+1) n)
    plus acor (r), ewt, yq, acor (w) (32n); every q+1 steps the PREPARE_NEXT norms read acor, ewt,
    zn[q], zn[qmax] (32n)."""
    n = CONFIGS[cfg][2]
    att = st["nst"] + st["netf"] + st["ncfn"]
    visits = st["nfe"] + st["nsetups"]
    return (visits * 2 * TS_RECORD_BYTES + st["nfe"] * (32 * n + 4) + st["nni"] * (8 * n * n + 12 * n + 48 * n) +
            att * (16 * (QBAR + 1) * n + 32 * n) + st["nst"] * 32 * n // (QBAR + 1))


def hbm_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except Exception:
        return 7700.0, "fallback: B200 nominal HBM3e 7.7 TB/s"


def traffic_split(cfg, st):
    """K_ctl DRAM bytes (read + write) per integrate, scaled per slot visit from the committed ncu --set full
    capture of one K_ctl launch (profiles/traffic.json "split_ctl": dram bytes / slots visited)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            t = json.load(f)["split_ctl_" + cfg]
        return t["dram_bytes_per_visit"] * (st["nfe"] + st["nsetups"])
    except Exception:
        return None


def traffic_per_launch(cfg, cells):
    """DRAM bytes (read + write) per launch, scaled per cell from the committed ncu --set full capture
    (profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum of one capture / its cells)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            t = json.load(f)[cfg]
        return t["dram_bytes_per_cell"] * cells
    except Exception:
        return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu):
        self.gpu, self.rows, self.p = gpu, [], None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = [r for r in self.rows if len(r) == len(self.FIELDS)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in rows:
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], r[4:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# ------------------------------------------------------------------ CPU oracle
def host_cpu():
    """CPU model, logical cores and SMT state of the host that runs the oracle baseline."""
    model, smt = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        smt = open("/sys/devices/system/cpu/smt/active").read().strip() == "1"
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count(), "smt_active": smt}


def oracle_cells_per_s(cfg, budget_s=15.0, threads=None, rank_cells=None, steps=1, dt=None, solver=None):
    """Time the CPU oracle (as it stands) on a bounded uniform random sample of the workload's cells
    (an unbiased estimate of the per-cell cost).  solver: oracle options (ls, maxl, method)."""
    from oracle import oracle as O
    model, mech, n, L, dt0, rtol, atol, _ = CONFIGS[cfg]
    dt = dt or dt0
    solver = solver or {}
    threads = threads or os.cpu_count() or 1
    if cfg in GLOBAL_CFGS:
        # the lockstep batch is one system: the oracle's global variant on a contiguous sub-batch, 1 thread
        from synth import flame_field
        om = O.Model.mechanism(mech)

        def runb(m):
            y, rho, F, _ = flame_field(mech, L, cells=np.arange(m), dt=dt)
            t = time.perf_counter()
            O.integrate_global(om, y, 0.0, dt, rtol, atol, rho=rho, fext_yc=F)
            return time.perf_counter() - t

        tp = runb(256)
        m = int(max(256, min(L ** 3, 256 * budget_s / max(tp, 1e-6))) // 256 * 256)
        return m, [runb(m) for _ in range(steps)], 1
    if cfg == "C1":
        y, rho, F, prog = make_inputs(cfg)
        om, G, idx = O.Model.robertson(), 1, np.arange(y.shape[1])
    elif cfg == "C2":
        from synth import nyx_field
        idx = np.sort(np.random.default_rng(0).choice(L ** 3, 65536, replace=False))
        e, rho, fe = nyx_field(L, cells=idx, dt=dt)
        y, F, om, G = e, fe, O.Model.nyx_kwh(), 1
        idx = np.arange(len(idx))
    else:
        from synth import flame_field
        # a uniform random sample of the grid's cells (seeded): the workload's own mix of fresh, reacting and
        # burnt cells
        # (~3-4 s per pass of the oracle on 16 host cores for the H2 / DRM19 fields; the 53-species ones are slower)
        nsamp = 120000 if cfg in ("C3", "C4") else 40000
        pick = np.sort(np.random.default_rng(2405017130).choice(L ** 3, min(L ** 3, nsamp), replace=False))
        y, rho, F, _ = flame_field(mech, L, cells=pick, dt=dt)
        om, G = O.Model.mechanism(mech), CONFIGS_G[cfg]
        idx = np.arange(len(pick))

    def run(sel):
        t = time.perf_counter()
        O.integrate_batch(om, y[:, sel], 0.0, dt, rtol, atol, rho=None if rho is None else rho[sel],
                          fext_yc=None if F is None else F[:, sel], group=G, threads=threads, **solver)
        return time.perf_counter() - t

    probe = idx[: min(len(idx), 512)]
    tp = run(probe)
    m = int(min(len(idx), max(len(probe), len(probe) * budget_s / max(tp, 1e-6))))
    sel = idx[np.linspace(0, len(idx) - 1, m).astype(int)]
    times = [run(sel) for _ in range(steps)]
    return m, times, threads


CONFIGS_G = {"C3": 1, "C4": 1, "C5P": 1}     # WRMS summation group of the default (thread-per-cell) kernel, R15


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, default=0, help="override cells per rank (debug; implies weak scaling)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's fixed grid dealt over the ranks in block-cyclic 16^3 tiles "
                         "(BASELINE: 256^3 sharded over 2/4/8 GPUs); weak: one full grid per rank")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--kernel", default=None, choices=["thread", "group", "split"],
                    help="per-cell kernel organisation of the mechanism models (default: the library's)")
    ap.add_argument("--jac", default="analytic", choices=["analytic", "dq"],
                    help="Jacobian: analytic (2A/2B) or CVODE's difference quotient (3A/3B; SPLIT kernel)")
    ap.add_argument("--ls", default="dense", choices=["dense", "diag", "gmres"],
                    help="Newton linear solver: dense LU (2A/3A), CVDiag (P:480) or GMRES (1A; SPLIT kernel)")
    ap.add_argument("--maxl", type=int, default=0, help="GMRES Krylov cap (0 = 5)")
    ap.add_argument("--method", default="bdf", choices=["bdf", "erk4"],
                    help="bdf (default) or the explicit adaptive ERK of P:415-426")
    ap.add_argument("--dt", type=float, default=0.0, help="override the config's dt_CFD")
    args = ap.parse_args()

    from paper_2405_01713_b200 import parallel as PL
    rank, world, local = PL.env_rank()
    cfg = args.config
    model, mech, n, L, dt, rtol, atol, desc = CONFIGS[cfg]
    if args.dt:
        desc = desc.replace("dt_CFD %g s" % dt, "dt_CFD %g s" % args.dt)
        dt = args.dt
    from oracle import oracle as _O   # constants only (solver ids); the product path never calls it
    solver = {}
    if args.ls != "dense":
        solver.update(ls={"diag": _O.LS_DIAG, "gmres": _O.LS_GMRES}[args.ls], maxl=args.maxl)
        desc += ", %s linear solver" % {"diag": "CVDiag", "gmres": "GMRES (inexact Newton-Krylov, 1A)"}[args.ls]
    if args.method == "erk4":
        solver.update(method=_O.METHOD_ERK4, mxstep=1000000)
        desc += ", explicit ERK 4(3) (P:415-426)"

    if args.impl == "reference":
        if rank != 0:
            return
        m, times, thr = oracle_cells_per_s(cfg, budget_s=max(5.0, 60.0 / max(args.steps, 1)), steps=args.warmup +
                                           args.steps, dt=dt, solver=solver)
        times = times[args.warmup:] or times
        tt = sum(times)
        val = m * len(times) / tt
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tt / len(times),
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": desc, "sample_cells_per_step": m},
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": thr, "kind": "oracle",
                                 "sample": (f"first {m} cells of the {cfg} field as one lockstep batch per step"
                                            if cfg in GLOBAL_CFGS else
                                            f"{m} uniformly sampled cells of the {cfg} workload per step"),
                                 "host": host_cpu()},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2405_01713_b200 as P

    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    scaling = "weak" if (args.cells or cfg in ("C5", "C5P")) else args.scaling
    y0, rho, F, prog = make_inputs(cfg, rank, args.cells or None, world, scaling)
    N = y0.shape[1]
    glob_mode = cfg in GLOBAL_CFGS
    b = P.Batch(N, n, rtol, atol, device=local, mode=P.MODE_GLOBAL_NORM if glob_mode else P.MODE_PER_CELL,
                mxstep=1000000 if args.method == "erk4" else 10000)
    if args.kernel and mech:
        b.set_kernel(args.kernel)
    b.set_model(model)
    if args.jac != "analytic":
        b.set_jacobian(args.jac)
    if args.ls != "dense":
        b.set_linear_solver(args.ls, args.maxl)
    if args.method != "bdf":
        b.set_method(args.method)
    if glob_mode and world > 1:
        # one lockstep system across ranks: the library's own NCCL communicator carries the norms
        uid = torch.cuda.nccl.unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        b.set_comm(obj[0], world, rank, rank_cells(cfg, rank, world, scaling, args.cells or None)[1])
    y_pristine = torch.tensor(y0, device=dev)
    y = torch.empty_like(y_pristine)
    Fd = None if F is None else torch.tensor(F, device=dev)
    rd = None if rho is None else torch.tensor(rho, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        b.integrate(0.0, dt, y, f_ext=Fd, aux=rd)

    for _ in range(args.warmup):
        y.copy_(y_pristine)
        step()
    torch.cuda.synchronize()
    st_w = b.stats()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kern_ms, stats, phase_ms = [], [], []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            y.copy_(y_pristine)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            torch.cuda.synchronize()
            kern_ms.append(b.last_kernel_ms())
            stats.append(b.stats())
            phase_ms.append(b.phase_ms())
    step_ms = [a.elapsed_time(z) for a, z in ev]
    total_ms = PL.max_over_ranks(sum(step_ms), dist, dev)
    ms_per_step = total_ms / args.steps
    n_total = int(PL.sum_over_ranks(N, dist, dev))
    value = n_total / (ms_per_step * 1e-3)

    # roofline: the binding roof of the per-cell path is the FP64 pipe; achieved = ALGORITHMIC
    # FP64 flops (unit_flops x per-cell statistics) / the kernel's event-timed duration on the launch stream.
    peak = SMS * FP64_FMA_PER_SM_CLK * 2 * SM_MAX_MHZ * 1e6 / 1e12
    probe = None
    try:
        import ctypes as C
        tf, sm = C.c_double(), C.c_int32()
        with ClockSampler(local) as pclk:
            ok = P._lib.lib().bdfb_probe_fp64(local, 500.0, C.byref(tf), C.byref(sm)) == 0
        if ok:
            probe = {"tflops": tf.value, "sms": sm.value, "clocks": pclk.summary(),
                     "kernel": "fp64_probe_kernel (8 independent DFMA chains per thread, all SMs)"}
    except Exception:
        pass
    tw = transc_weights()
    pf = [phase_flops(cfg, s, args.method, args.ls) for s in stats]
    flops = [sum(p.values()) for p in pf]
    whole = statistics.mean(f / (k * 1e-3) for f, k in zip(flops, kern_ms)) / 1e12
    roof_common = {"bound": "alu", "pipe": "fp64", "peak": peak, "unit": "TFLOP/s",
                   "peak_source": "derived from B200_PROFILING.md unit counts: 148 SM x 64 FP64 FMA/clk x 2 x 1965 "
                                  "MHz (MEASURED_PEAKS.json has no FP64 entry); fp64_probe is the measured DFMA "
                                  "throughput with its clocks",
                   "fp64_probe": probe, "transcendental_flops": tw,
                   "whole_step": {"achieved": whole, "frac": whole / peak, "flops_per_integrate": statistics.mean(flops),
                                  "ms": statistics.mean(kern_ms)}}
    kname = (("integrate_tpc_kernel<Tpc_%s>" if b.wrms_group == 1 else "integrate_group_kernel<ModelMech<%s>>")
             % mech) if mech else "integrate_kernel<%s>" % model
    if args.method == "erk4":
        kname = "erk_kernel<Tpc_%s>" % mech
    roof = dict(roof_common, achieved=whole, frac=whole / peak, traffic=traffic_per_launch(cfg, N), kernel=kname,
                kernel_ms=statistics.mean(kern_ms), flops_per_launch=statistics.mean(flops))
    phases = None
    if phase_ms and phase_ms[0]:
        # SPLIT: four kernels per trip, timed per phase with CUDA events on the launch stream.  The roofline is
        # the dominant kernel's algorithmic FP64 fraction; the whole-step fraction sits beside it; K_ctl's HBM
        # traffic (its slot-state round trips, an implementation cost, not algorithmic bytes) is a diagnostic.
        hpk, src = hbm_peak()
        pm = {k: statistics.mean(p[k] for p in phase_ms) for k in phase_ms[0]}
        tot = sum(pm.values())
        phases = {}
        for k, v in pm.items():
            fl = statistics.mean(p[k] for p in pf)
            tfl = fl / (v * 1e-3) / 1e12 if v > 0 else 0.0
            phases[k] = {"ms": v, "share": v / tot, "flops": fl, "tflops": tfl, "frac": tfl / peak}
        cb = statistics.mean(ctl_bytes(cfg, s) for s in stats)
        phases["ctl"]["hbm_model"] = {"bytes": cb, "gbs": cb / (pm["ctl"] * 1e-3) / 1e9,
                                      "frac": cb / (pm["ctl"] * 1e-3) / 1e9 / hpk, "peak_source": src,
                                      "traffic_ncu": traffic_split(cfg, stats[-1]),
                                      "model": "DESIGN.md §6 (slot-state round trips: implementation bytes)"}
        dom = max(pm, key=pm.get)
        big = n > 32   # split_big.cuh setup kernels
        knames = {"ctl": "erk_ctl_kernel" if args.method == "erk4" else "split_ctl_kernel",
                  "jac": "split_jac_lanes_kernel" if big else "split_jac_kernel",
                  "lu": "split_lu_rows_kernel" if big else "split_lu_kernel", "rhs": "split_rhs_kernel"}
        roof = dict(roof_common, achieved=phases[dom]["tflops"], frac=phases[dom]["frac"],
                    traffic=traffic_split(cfg, stats[-1]) if dom == "ctl" else None,
                    kernel=f"{knames[dom]}<Tpc_{mech}> (K_{dom}, {100 * pm[dom] / tot:.0f}% of the step)",
                    kernel_ms=pm[dom], flops_per_launch=phases[dom]["flops"])
    if glob_mode:
        # lockstep batch: the state, J and LU stream through HBM every stage -> HBM roofline
        hb = [hbm_bytes_global(cfg, s) for s in stats]
        gbs = statistics.mean(x / (k * 1e-3) for x, k in zip(hb, kern_ms)) / 1e9
        hpk, src = hbm_peak()
        roof = {"bound": "hbm", "achieved": gbs, "peak": hpk, "unit": "GB/s", "frac": gbs / hpk,
                "traffic": traffic_per_launch(cfg, N), "kernel": "global-norm kernel sequence (gk_*)",
                "peak_source": src, "kernel_ms": statistics.mean(kern_ms),
                "bytes_per_integrate": statistics.mean(hb), "fp64": roof_common}

    # e2e through the host-buffer C-ABI call (pinned host memory; H2D + integrate + D2H timed)
    yh0 = torch.tensor(y0).pin_memory()
    yh = torch.empty_like(yh0).pin_memory()
    Fh = None if F is None else torch.tensor(F).pin_memory()
    rh = None if rho is None else torch.tensor(rho).pin_memory()
    yh.copy_(yh0)
    b.integrate_host(0.0, dt, yh, f_ext=Fh, aux=rh)            # allocates the staging buffers (warm-up)
    e2e_ms = []
    for i in range(args.steps):
        yh.copy_(yh0)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        b.integrate_host(0.0, dt, yh, f_ext=Fh, aux=rh)
        z.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(a.elapsed_time(z))
    e2e_total = PL.max_over_ranks(sum(e2e_ms), dist, dev)
    h2d = y0.nbytes + (0 if F is None else F.nbytes) + (0 if rho is None else rho.nbytes)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        m, times, thr = oracle_cells_per_s(cfg, budget_s=5.0, dt=dt, solver=solver, steps=3)
        smp = (f"first {m} cells of the {cfg} field integrated as one lockstep batch (orc_integrate_global)"
               if glob_mode else f"{m} uniformly sampled cells of the {cfg} workload (same recipe and seed)")
        smp += f"; median of {len(times)} passes (Python threads calling the C oracle, GIL released)"
        cpu = {"value": m / statistics.median(times), "unit": UNIT, "cores": thr, "kind": "oracle", "sample": smp,
               "passes_s": times, "host": host_cpu()}

    s = PL.reduce_stats(stats[-1], dist, dev)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "cells_total": n_total, "cells_per_gpu": N, "n": n, "rtol": rtol,
                           "atol": atol if np.isscalar(atol) else list(atol), "dt_CFD": dt,
                           "mode": "global-norm" if glob_mode else "per-cell",
                           "parallelism": (f"dp{world} (cells sharded; NCCL allgather of the batch norms)"
                                           if glob_mode else f"dp{world} (cells sharded, no collective)"),
                           "partition": ("single GPU" if world == 1 else
                                         "contiguous slabs" if (cfg == "C1" or glob_mode or scaling == "weak") else
                                         "block-cyclic 16^3 tiles"),
                           "l2": "inputs larger than L2 (state %.2f GB per GPU); pristine field restored "
                                 "untimed before each step" % (y0.nbytes / 1e9),
                           "mechanism": mech, "jacobian": args.jac, "linear_solver": args.ls,
                           "method": args.method},
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": n_total / (e2e_total / args.steps * 1e-3), "unit": UNIT,
                        "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(y0.nbytes)},
                "gpu_launches": args.steps * b.last_launch_count(),
                "clocks": clk.summary(),
                "stats": {k: s[k] for k in ("n_cells", "n_failed", "nst", "nfe", "nje", "nsetups", "nni", "netf",
                                            "ncfn", "nst_max", "nli") if k in s},
                "kernel_ms_per_step": kern_ms, "phases": phases}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
