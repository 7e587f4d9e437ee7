"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

Holds NONE of the method's arithmetic: only counter-based random numbers
(SplitMix64 keyed by (seed, cell, field)), smooth Fourier fields on an L^3
grid, and the per-config field recipes of SURVEY.md §8(d).1 / DESIGN.md
"Input recipe".  Because every value is a pure function of (seed, global
cell index, field id), any rank can generate any subset of cells and the
field is identical under every sharding.

The reacting-cell states of the flame template are read from
synth/data/<mech>_trajectory.npz, written once by synth/make_trajectories.py
(which integrates a 0-D reactor with the CPU oracle only).
"""
from .fields import (SEED_BASE, autoignition_box, config_seed, flame_field, gaussian, nyx_field, robertson_field, splitmix64,
                     uniform)

__all__ = ["SEED_BASE", "autoignition_box", "config_seed", "splitmix64", "uniform", "gaussian", "robertson_field", "nyx_field",
           "flame_field"]
