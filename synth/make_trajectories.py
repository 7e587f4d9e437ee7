"""Write synth/data/<mech>_trajectory.npz: a 0-D constant-volume ignition
trajectory from the fresh mixture at T_u, 1 atm,
integrated with the CPU ORACLE ONLY at rtol = 1e-10.  States are tabulated
against the normalised temperature rise c = (T - T_u)/(T_b - T_u) for the
flame-field template's reacting cells.  Run once; the output is committed.

    python synth/make_trajectories.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle as O  # noqa: E402
from synth.fields import MIXTURES, fresh_state  # noqa: E402


def trajectory(mech, points=400):
    m = O.Model.mechanism(mech)
    Yf, W, T_cold, T_u, rho_u = fresh_state(mech)
    y = np.concatenate([Yf, [T_u]])
    ts = np.concatenate([[0.0], np.logspace(-8, 0, 400)])
    out = [y.copy()]
    t_prev = 0.0
    for t1 in ts[1:]:
        # subdivide an interval until the temperature rise per output is < 0.5 % of the total
        stack = [t1]
        while stack:
            tt = stack[-1]
            y1, st, _ = O.integrate(m, y, t_prev, tt, 1e-10, 1e-20, rho_u, mxstep=200000)
            assert st["status"] == 0, st
            if abs(y1[-1] - y[-1]) > 10.0 and tt - t_prev > 1e-12:
                stack.append(0.5 * (t_prev + tt))
                continue
            stack.pop()
            y, t_prev = y1, tt
            out.append(y.copy())
    S = np.array(out)
    T = S[:, -1]
    Tb = T[-1]
    c = (T - T_u) / (Tb - T_u)
    c = np.maximum.accumulate(c)
    grid = np.linspace(0.0, 1.0, points)
    # monotone in time until burnt: sample states at the first crossing of each grid value
    idx = np.searchsorted(c, grid, side="left").clip(0, len(c) - 1)
    states = S[idx]
    states[-1] = S[-1]
    cg = c[idx]
    cg[0], cg[-1] = 0.0, 1.0
    keep = np.concatenate([[True], np.diff(cg) > 0])
    return cg[keep], states[keep], rho_u, Tb


def main(argv=None):
    os.makedirs(os.path.join(HERE, "data"), exist_ok=True)
    argv = sys.argv[1:] if argv is None else argv
    for mech in (argv or MIXTURES):
        c, s, rho, Tb = trajectory(mech)
        np.savez_compressed(os.path.join(HERE, "data", f"{mech}_trajectory.npz"), c=c, states=s, rho=rho, Tb=Tb)
        print(mech, "points", len(c), "T_b", Tb, "rho", rho)


if __name__ == "__main__":
    main()
