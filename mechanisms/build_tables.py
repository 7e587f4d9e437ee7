"""Write the mechanism tables mechanisms/*.json (problem DATA, not method code).

The paper names its mechanisms only by size (DRM21/DOD53/HEP88; a
53-species n-dodecane) and none ships with /root/reference; this
sandbox has no network (reading R22).  The tables below are
therefore *class-equivalent* mechanisms, restated from memory of the public
GRI-Mech 3.0 / Li et al. (2004) rate and thermo data, not copies of the
published files:

* ``h2_lidryer``  -- 9 species + T (n = 10), 21 reactions, Li-Dryer-class
  H2/O2/N2 (config C3).
* ``drm19_class`` -- 21 species + T (n = 22), 84 reactions, DRM19-class
  CH4/air built from GRI-3.0-style expressions over the DRM19 species set
  (config C4).

Checks run on every build (a failure aborts): every reaction is element
balanced; every NASA-7 pair is continuous at Tmid in cp/R, h/RT and s/R
(this catches mis-remembered coefficients); standard enthalpies of formation
of a few species match textbook values.

Usage: python mechanisms/build_tables.py      (rewrites the .json files)
"""
from __future__ import annotations

import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))

ATOMIC = {"H": 1.00794, "O": 15.9994, "C": 12.0107, "N": 14.0067, "AR": 39.948}

# ---- thermo: NASA-7, Tmid = 1000 K (GRI-Mech 3.0 style, restated) --------
THERMO = {
    "H2": ({"H": 2},
           [2.34433112e+00, 7.98052075e-03, -1.94781510e-05, 2.01572094e-08, -7.37611761e-12, -9.17935173e+02, 6.83010238e-01],
           [3.33727920e+00, -4.94024731e-05, 4.99456778e-07, -1.79566394e-10, 2.00255376e-14, -9.50158922e+02, -3.20502331e+00]),
    "H": ({"H": 1},
          [2.50000000e+00, 7.05332819e-13, -1.99591964e-15, 2.30081632e-18, -9.27732332e-22, 2.54736599e+04, -4.46682853e-01],
          [2.50000001e+00, -2.30842973e-11, 1.61561948e-14, -4.73515235e-18, 4.98197357e-22, 2.54736599e+04, -4.46682914e-01]),
    "O": ({"O": 1},
          [3.16826710e+00, -3.27931884e-03, 6.64306396e-06, -6.12806624e-09, 2.11265971e-12, 2.91222592e+04, 2.05193346e+00],
          [2.56942078e+00, -8.59741137e-05, 4.19484589e-08, -1.00177799e-11, 1.22833691e-15, 2.92175791e+04, 4.78433864e+00]),
    "O2": ({"O": 2},
           [3.78245636e+00, -2.99673416e-03, 9.84730201e-06, -9.68129509e-09, 3.24372837e-12, -1.06394356e+03, 3.65767573e+00],
           [3.28253784e+00, 1.48308754e-03, -7.57966669e-07, 2.09470555e-10, -2.16717794e-14, -1.08845772e+03, 5.45323129e+00]),
    "OH": ({"O": 1, "H": 1},
           [3.99201543e+00, -2.40131752e-03, 4.61793841e-06, -3.88113333e-09, 1.36411470e-12, 3.61508056e+03, -1.03925458e-01],
           [3.09288767e+00, 5.48429716e-04, 1.26505228e-07, -8.79461556e-11, 1.17412376e-14, 3.85865700e+03, 4.47669610e+00]),
    "H2O": ({"H": 2, "O": 1},
            [4.19864056e+00, -2.03643410e-03, 6.52040211e-06, -5.48797062e-09, 1.77197817e-12, -3.02937267e+04, -8.49032208e-01],
            [3.03399249e+00, 2.17691804e-03, -1.64072518e-07, -9.70419870e-11, 1.68200992e-14, -3.00042971e+04, 4.96677010e+00]),
    "HO2": ({"H": 1, "O": 2},
            [4.30179801e+00, -4.74912051e-03, 2.11582891e-05, -2.42763894e-08, 9.29225124e-12, 2.94808040e+02, 3.71666245e+00],
            [4.01721090e+00, 2.23982013e-03, -6.33658150e-07, 1.14246370e-10, -1.07908535e-14, 1.11856713e+02, 3.78510215e+00]),
    "H2O2": ({"H": 2, "O": 2},
             [4.27611269e+00, -5.42822417e-04, 1.67335701e-05, -2.15770813e-08, 8.62454363e-12, -1.77025821e+04, 3.43505074e+00],
             [4.16500285e+00, 4.90831694e-03, -1.90139225e-06, 3.71185986e-10, -2.87908305e-14, -1.78617877e+04, 2.91615662e+00]),
    "CH2": ({"C": 1, "H": 2},
            [3.76267867e+00, 9.68872143e-04, 2.79489841e-06, -3.85091153e-09, 1.68741719e-12, 4.60040401e+04, 1.56253185e+00],
            [2.87410113e+00, 3.65639292e-03, -1.40894597e-06, 2.60179549e-10, -1.87727567e-14, 4.62636040e+04, 6.17119324e+00]),
    "CH2(S)": ({"C": 1, "H": 2},
               [4.19860411e+00, -2.36661419e-03, 8.23296220e-06, -6.68815981e-09, 1.94314737e-12, 5.04968163e+04, -7.69118967e-01],
               [2.29203842e+00, 4.65588637e-03, -2.01191947e-06, 4.17906000e-10, -3.39716365e-14, 5.09259997e+04, 8.62650169e+00]),
    "CH3": ({"C": 1, "H": 3},
            [3.67359040e+00, 2.01095175e-03, 5.73021856e-06, -6.87117425e-09, 2.54385734e-12, 1.64449988e+04, 1.60456433e+00],
            [2.28571772e+00, 7.23990037e-03, -2.98714348e-06, 5.95684644e-10, -4.67154394e-14, 1.67755843e+04, 8.48007179e+00]),
    "CH4": ({"C": 1, "H": 4},
            [5.14987613e+00, -1.36709788e-02, 4.91800599e-05, -4.84743026e-08, 1.66693956e-11, -1.02466476e+04, -4.64130376e+00],
            [7.48514950e-02, 1.33909467e-02, -5.73285809e-06, 1.22292535e-09, -1.01815230e-13, -9.46834459e+03, 1.84373180e+01]),
    "CO": ({"C": 1, "O": 1},
           [3.57953347e+00, -6.10353680e-04, 1.01681433e-06, 9.07005884e-10, -9.04424499e-13, -1.43440860e+04, 3.50840928e+00],
           [2.71518561e+00, 2.06252743e-03, -9.98825771e-07, 2.30053008e-10, -2.03647716e-14, -1.41518724e+04, 7.81868772e+00]),
    "CO2": ({"C": 1, "O": 2},
            [2.35677352e+00, 8.98459677e-03, -7.12356269e-06, 2.45919022e-09, -1.43699548e-13, -4.83719697e+04, 9.90105222e+00],
            [3.85746029e+00, 4.41437026e-03, -2.21481404e-06, 5.23490188e-10, -4.72084164e-14, -4.87591660e+04, 2.27163806e+00]),
    "HCO": ({"H": 1, "C": 1, "O": 1},
            [4.22118584e+00, -3.24392532e-03, 1.37799446e-05, -1.33144093e-08, 4.33768865e-12, 3.83956496e+03, 3.39437243e+00],
            [2.77217438e+00, 4.95695526e-03, -2.48445613e-06, 5.89161778e-10, -5.33508711e-14, 4.01191815e+03, 9.79834492e+00]),
    "CH2O": ({"H": 2, "C": 1, "O": 1},
             [4.79372315e+00, -9.90833369e-03, 3.73220008e-05, -3.79285261e-08, 1.31772652e-11, -1.43089567e+04, 6.02812900e-01],
             [1.76069008e+00, 9.20000082e-03, -4.42258813e-06, 1.00641212e-09, -8.83855640e-14, -1.39958323e+04, 1.36563230e+01]),
    "CH3O": ({"C": 1, "H": 3, "O": 1},
             [2.10620400e+00, 7.21659500e-03, 5.33847200e-06, -7.37763600e-09, 2.07561000e-12, 9.78601100e+02, 1.31521770e+01],
             [3.77079900e+00, 7.87149700e-03, -2.65638400e-06, 3.94443100e-10, -2.11261600e-14, 1.27832520e+02, 2.92957500e+00]),
    "C2H4": ({"C": 2, "H": 4},
             [3.95920148e+00, -7.57052247e-03, 5.70990292e-05, -6.91588753e-08, 2.69884373e-11, 5.08977593e+03, 4.09733096e+00],
             [2.03611116e+00, 1.46454151e-02, -6.71077915e-06, 1.47222923e-09, -1.25706061e-13, 4.93988614e+03, 1.03053693e+01]),
    "C2H5": ({"C": 2, "H": 5},
             [4.30646568e+00, -4.18658892e-03, 4.97142807e-05, -5.99126606e-08, 2.30509004e-11, 1.28416265e+04, 4.70720924e+00],
             [1.95465642e+00, 1.73972722e-02, -7.98206668e-06, 1.75217689e-09, -1.49641576e-13, 1.28575200e+04, 1.34624343e+01]),
    "C2H6": ({"C": 2, "H": 6},
             [4.29142492e+00, -5.50154270e-03, 5.99438288e-05, -7.08466285e-08, 2.68685771e-11, -1.15222055e+04, 2.66682316e+00],
             [1.07188150e+00, 2.16852677e-02, -1.00256067e-05, 2.21412001e-09, -1.90002890e-13, -1.14263932e+04, 1.51156107e+01]),
    "N2": ({"N": 2},
           [3.29867700e+00, 1.40824040e-03, -3.96322200e-06, 5.64151500e-09, -2.44485400e-12, -1.02089990e+03, 3.95037200e+00],
           [2.92664000e+00, 1.48797680e-03, -5.68476000e-07, 1.00970380e-10, -6.75335100e-15, -9.22797700e+02, 5.98052800e+00]),
    "AR": ({"AR": 1},
           [2.5, 0.0, 0.0, 0.0, 0.0, -7.45375000e+02, 4.36600000e+00],
           [2.5, 0.0, 0.0, 0.0, 0.0, -7.45375000e+02, 4.36600000e+00]),
}

# ---- reactions ------------------------------------------------------------
# (equation, A [cm,mol,s], b, Ea [cal/mol], extras)
# extras: type = 'tb' (three body, +M), 'lind' / 'troe' (falloff (+M)),
#         low = (A0, b0, Ea0), troe = (a, T3, T1[, T2]), eff = {species: alpha}

H2_STD = {"H2": 2.5, "H2O": 12.0}
H2_REACTIONS = [
    ("H + O2 <=> O + OH", 3.547e15, -0.406, 1.6599e4, {}),
    ("O + H2 <=> H + OH", 0.508e5, 2.67, 0.629e4, {}),
    ("H2 + OH <=> H2O + H", 0.216e9, 1.51, 0.343e4, {}),
    ("O + H2O <=> OH + OH", 2.97e6, 2.02, 1.34e4, {}),
    ("H2 + M <=> H + H + M", 4.577e19, -1.40, 1.0438e5, {"type": "tb", "eff": H2_STD}),
    ("O + O + M <=> O2 + M", 6.165e15, -0.50, 0.0, {"type": "tb", "eff": H2_STD}),
    ("O + H + M <=> OH + M", 4.714e18, -1.00, 0.0, {"type": "tb", "eff": H2_STD}),
    ("H + OH + M <=> H2O + M", 3.800e22, -2.00, 0.0, {"type": "tb", "eff": H2_STD}),
    ("H + O2 (+M) <=> HO2 (+M)", 1.475e12, 0.60, 0.0,
     {"type": "troe", "low": (6.366e20, -1.72, 5.248e2), "troe": (0.8, 1e-30, 1e30),
      "eff": {"H2": 2.0, "H2O": 11.0, "O2": 0.78}}),
    ("HO2 + H <=> H2 + O2", 1.66e13, 0.0, 0.823e3, {}),
    ("HO2 + H <=> OH + OH", 7.079e13, 0.0, 2.95e2, {}),
    ("HO2 + O <=> O2 + OH", 0.325e14, 0.0, 0.0, {}),
    ("HO2 + OH <=> H2O + O2", 2.890e13, 0.0, -4.970e2, {}),
    ("HO2 + HO2 <=> H2O2 + O2", 4.200e14, 0.0, 1.1982e4, {}),
    ("HO2 + HO2 <=> H2O2 + O2", 1.300e11, 0.0, -1.6293e3, {}),
    ("H2O2 (+M) <=> OH + OH (+M)", 2.951e14, 0.0, 4.843e4,
     {"type": "troe", "low": (1.202e17, 0.0, 4.55e4), "troe": (0.5, 1e-30, 1e30), "eff": H2_STD}),
    ("H2O2 + H <=> H2O + OH", 0.241e14, 0.0, 0.397e4, {}),
    ("H2O2 + H <=> HO2 + H2", 0.482e14, 0.0, 0.795e4, {}),
    ("H2O2 + O <=> OH + HO2", 9.550e6, 2.00, 3.970e3, {}),
    ("H2O2 + OH <=> HO2 + H2O", 1.000e12, 0.0, 0.0, {}),
    ("H2O2 + OH <=> HO2 + H2O", 5.800e14, 0.0, 9.557e3, {}),
]

STD = {"H2": 2.0, "H2O": 6.0, "CH4": 2.0, "CO": 1.5, "CO2": 2.0, "C2H6": 3.0, "AR": 0.7}
STD_NOAR = {k: v for k, v in STD.items() if k != "AR"}
DRM_REACTIONS = [
    ("O + O + M <=> O2 + M", 1.200e17, -1.0, 0.0,
     {"type": "tb", "eff": {"H2": 2.4, "H2O": 15.4, "CH4": 2.0, "CO": 1.75, "CO2": 3.6, "C2H6": 3.0, "AR": 0.83}}),
    ("O + H + M <=> OH + M", 5.000e17, -1.0, 0.0, {"type": "tb", "eff": STD}),
    ("O + H2 <=> H + OH", 3.870e4, 2.70, 6260.0, {}),
    ("O + HO2 <=> OH + O2", 2.000e13, 0.0, 0.0, {}),
    ("O + CH2 <=> H + HCO", 8.000e13, 0.0, 0.0, {}),
    ("O + CH2(S) <=> H + HCO", 1.500e13, 0.0, 0.0, {}),
    ("O + CH3 <=> H + CH2O", 5.060e13, 0.0, 0.0, {}),
    ("O + CH4 <=> OH + CH3", 1.020e9, 1.50, 8600.0, {}),
    ("O + CO (+M) <=> CO2 (+M)", 1.800e10, 0.0, 2385.0,
     {"type": "lind", "low": (6.020e14, 0.0, 3000.0),
      "eff": {"H2": 2.0, "O2": 6.0, "H2O": 6.0, "CH4": 2.0, "CO": 1.5, "CO2": 3.5, "C2H6": 3.0, "AR": 0.5}}),
    ("O + HCO <=> OH + CO", 3.000e13, 0.0, 0.0, {}),
    ("O + HCO <=> H + CO2", 3.000e13, 0.0, 0.0, {}),
    ("O + CH2O <=> OH + HCO", 3.900e13, 0.0, 3540.0, {}),
    ("O + C2H4 <=> CH3 + HCO", 1.250e7, 1.83, 220.0, {}),
    ("O + C2H5 <=> CH3 + CH2O", 2.240e13, 0.0, 0.0, {}),
    ("O + C2H6 <=> OH + C2H5", 8.980e7, 1.92, 5690.0, {}),
    ("O2 + CO <=> O + CO2", 2.500e12, 0.0, 47800.0, {}),
    ("O2 + CH2O <=> HO2 + HCO", 1.000e14, 0.0, 40000.0, {}),
    ("H + O2 + M <=> HO2 + M", 2.800e18, -0.86, 0.0,
     {"type": "tb", "eff": {"O2": 0.0, "H2O": 0.0, "CO": 0.75, "CO2": 1.5, "C2H6": 1.5, "N2": 0.0, "AR": 0.0}}),
    ("H + O2 + O2 <=> HO2 + O2", 2.080e19, -1.24, 0.0, {}),
    ("H + O2 + H2O <=> HO2 + H2O", 1.126e19, -0.76, 0.0, {}),
    ("H + O2 + N2 <=> HO2 + N2", 2.600e19, -1.24, 0.0, {}),
    ("H + O2 + AR <=> HO2 + AR", 7.000e17, -0.80, 0.0, {}),
    ("H + O2 <=> O + OH", 2.650e16, -0.6707, 17041.0, {}),
    ("H + H + M <=> H2 + M", 1.000e18, -1.0, 0.0,
     {"type": "tb", "eff": {"H2": 0.0, "H2O": 0.0, "CH4": 2.0, "CO2": 0.0, "C2H6": 3.0, "AR": 0.63}}),
    ("H + H + H2 <=> H2 + H2", 9.000e16, -0.6, 0.0, {}),
    ("H + H + H2O <=> H2 + H2O", 6.000e19, -1.25, 0.0, {}),
    ("H + H + CO2 <=> H2 + CO2", 5.500e20, -2.0, 0.0, {}),
    ("H + OH + M <=> H2O + M", 2.200e22, -2.0, 0.0,
     {"type": "tb", "eff": {"H2": 0.73, "H2O": 3.65, "CH4": 2.0, "C2H6": 3.0, "AR": 0.38}}),
    ("H + HO2 <=> O + H2O", 3.970e12, 0.0, 671.0, {}),
    ("H + HO2 <=> O2 + H2", 4.480e13, 0.0, 1068.0, {}),
    ("H + HO2 <=> OH + OH", 8.400e13, 0.0, 635.0, {}),
    ("H + CH2 (+M) <=> CH3 (+M)", 6.000e14, 0.0, 0.0,
     {"type": "troe", "low": (1.040e26, -2.76, 1600.0), "troe": (0.5620, 91.0, 5836.0, 8552.0), "eff": STD}),
    ("H + CH3 (+M) <=> CH4 (+M)", 1.390e16, -0.534, 536.0,
     {"type": "troe", "low": (2.620e33, -4.76, 2440.0), "troe": (0.7830, 74.0, 2941.0, 6964.0),
      "eff": dict(STD, CH4=3.0)}),
    ("H + CH4 <=> CH3 + H2", 6.600e8, 1.62, 10840.0, {}),
    ("H + HCO (+M) <=> CH2O (+M)", 1.090e12, 0.48, -260.0,
     {"type": "troe", "low": (2.470e24, -2.57, 425.0), "troe": (0.7824, 271.0, 2755.0, 6570.0), "eff": STD}),
    ("H + HCO <=> H2 + CO", 7.340e13, 0.0, 0.0, {}),
    ("H + CH2O (+M) <=> CH3O (+M)", 5.400e11, 0.454, 2600.0,
     {"type": "troe", "low": (2.200e30, -4.80, 5560.0), "troe": (0.7580, 94.0, 1555.0, 4200.0), "eff": STD_NOAR}),
    ("H + CH2O <=> HCO + H2", 5.740e7, 1.90, 2742.0, {}),
    ("H + CH3O <=> OH + CH3", 1.500e12, 0.50, -110.0, {}),
    ("H + C2H4 (+M) <=> C2H5 (+M)", 5.400e11, 0.454, 1820.0,
     {"type": "troe", "low": (6.000e41, -7.62, 6970.0), "troe": (0.9753, 210.0, 984.0, 4374.0), "eff": STD}),
    ("H + C2H5 (+M) <=> C2H6 (+M)", 5.210e17, -0.99, 1580.0,
     {"type": "troe", "low": (1.990e41, -7.08, 6685.0), "troe": (0.8422, 125.0, 2219.0, 6882.0), "eff": STD}),
    ("H + C2H6 <=> C2H5 + H2", 1.150e8, 1.90, 7530.0, {}),
    ("H2 + CO (+M) <=> CH2O (+M)", 4.300e7, 1.50, 79600.0,
     {"type": "troe", "low": (5.070e27, -3.42, 84350.0), "troe": (0.9320, 197.0, 1540.0, 10300.0), "eff": STD}),
    ("OH + H2 <=> H + H2O", 2.160e8, 1.51, 3430.0, {}),
    ("OH + OH <=> O + H2O", 3.570e4, 2.40, -2110.0, {}),
    ("OH + HO2 <=> O2 + H2O", 1.450e13, 0.0, -500.0, {}),
    ("OH + CH2 <=> H + CH2O", 2.000e13, 0.0, 0.0, {}),
    ("OH + CH2(S) <=> H + CH2O", 3.000e13, 0.0, 0.0, {}),
    ("OH + CH3 <=> CH2 + H2O", 5.600e7, 1.60, 5420.0, {}),
    ("OH + CH3 <=> CH2(S) + H2O", 6.440e17, -1.34, 1417.0, {}),
    ("OH + CH4 <=> CH3 + H2O", 1.000e8, 1.60, 3120.0, {}),
    ("OH + CO <=> H + CO2", 4.760e7, 1.228, 70.0, {}),
    ("OH + HCO <=> H2O + CO", 5.000e13, 0.0, 0.0, {}),
    ("OH + CH2O <=> HCO + H2O", 3.430e9, 1.18, -447.0, {}),
    ("OH + C2H6 <=> C2H5 + H2O", 3.540e6, 2.12, 870.0, {}),
    ("HO2 + CH2 <=> OH + CH2O", 2.000e13, 0.0, 0.0, {}),
    ("HO2 + CH3 <=> O2 + CH4", 1.000e12, 0.0, 0.0, {}),
    ("HO2 + CH3 <=> OH + CH3O", 3.780e13, 0.0, 0.0, {}),
    ("HO2 + CO <=> OH + CO2", 1.500e14, 0.0, 23600.0, {}),
    ("CH2 + O2 <=> OH + H + CO", 5.000e12, 0.0, 1500.0, {}),
    ("CH2 + H2 <=> H + CH3", 5.000e5, 2.0, 7230.0, {}),
    ("CH2 + CH3 <=> H + C2H4", 4.000e13, 0.0, 0.0, {}),
    ("CH2 + CH4 <=> CH3 + CH3", 2.460e6, 2.0, 8270.0, {}),
    ("CH2(S) + N2 <=> CH2 + N2", 1.500e13, 0.0, 600.0, {}),
    ("CH2(S) + AR <=> CH2 + AR", 9.000e12, 0.0, 600.0, {}),
    ("CH2(S) + O2 <=> H + OH + CO", 2.800e13, 0.0, 0.0, {}),
    ("CH2(S) + O2 <=> CO + H2O", 1.200e13, 0.0, 0.0, {}),
    ("CH2(S) + H2 <=> CH3 + H", 7.000e13, 0.0, 0.0, {}),
    ("CH2(S) + H2O <=> CH2 + H2O", 3.000e13, 0.0, 0.0, {}),
    ("CH2(S) + CH3 <=> H + C2H4", 1.200e13, 0.0, -570.0, {}),
    ("CH2(S) + CH4 <=> CH3 + CH3", 1.600e13, 0.0, -570.0, {}),
    ("CH2(S) + CO2 <=> CH2O + CO", 1.400e13, 0.0, 0.0, {}),
    ("CH3 + O2 <=> O + CH3O", 3.560e13, 0.0, 30480.0, {}),
    ("CH3 + O2 <=> OH + CH2O", 2.310e12, 0.0, 20315.0, {}),
    ("CH3 + CH3 (+M) <=> C2H6 (+M)", 6.770e16, -1.18, 654.0,
     {"type": "troe", "low": (3.400e41, -7.03, 2762.0), "troe": (0.6190, 73.2, 1180.0, 9999.0), "eff": STD}),
    ("CH3 + CH3 <=> H + C2H5", 6.840e12, 0.10, 10600.0, {}),
    ("CH3 + HCO <=> CH4 + CO", 2.648e13, 0.0, 0.0, {}),
    ("CH3 + CH2O <=> HCO + CH4", 3.320e3, 2.81, 5860.0, {}),
    ("CH3 + C2H6 <=> C2H5 + CH4", 6.140e6, 1.74, 10450.0, {}),
    ("HCO + H2O <=> H + CO + H2O", 1.500e18, -1.0, 17000.0, {}),
    ("HCO + M <=> H + CO + M", 1.870e17, -1.0, 17000.0, {"type": "tb", "eff": dict(STD_NOAR, H2O=0.0)}),
    ("HCO + O2 <=> HO2 + CO", 1.345e13, 0.0, 400.0, {}),
    ("CH3O + O2 <=> HO2 + CH2O", 4.280e-13, 7.60, -3530.0, {}),
    ("C2H5 + O2 <=> HO2 + C2H4", 8.400e11, 0.0, 3875.0, {}),
]

MECHS = {
    "h2_lidryer": {
        "species": ["H2", "O2", "H2O", "H", "O", "OH", "HO2", "H2O2", "N2"],
        "reactions": H2_REACTIONS,
        "provenance": ("Li-Dryer-class H2/O2 mechanism (9 species, 21 reactions incl. duplicates) "
                       "restated from memory of Li, Zhao, Kazakov & Dryer, IJCK 36 (2004); "
                       "NASA-7 thermo restated from GRI-Mech 3.0.  Not the published file "
                       "(no network; SURVEY.md R22).  Parity does not depend on the source."),
    },
    "drm19_class": {
        "species": ["H2", "H", "O", "O2", "OH", "H2O", "HO2", "CH2", "CH2(S)", "CH3", "CH4",
                    "CO", "CO2", "HCO", "CH2O", "CH3O", "C2H4", "C2H5", "C2H6", "N2", "AR"],
        "reactions": DRM_REACTIONS,
        "provenance": ("DRM19-class CH4/air mechanism: the DRM19 species set (21 species) with 84 "
                       "reactions restated from memory of GRI-Mech 3.0 rate expressions; NASA-7 "
                       "thermo from GRI-Mech 3.0.  Class-equivalent (same K, reaction count and "
                       "type mix), not the published DRM19 file (SURVEY.md R22)."),
    },
}


def parse_side(side):
    toks = [t.strip() for t in side.replace("(+M)", "").split("+")]
    out, m = [], False
    for t in toks:
        if not t:
            continue
        if t == "M":
            m = True
            continue
        out.append(t)
    return out, m


def nasa_eval(a, T):
    cp = a[0] + a[1] * T + a[2] * T**2 + a[3] * T**3 + a[4] * T**4
    h = a[0] + a[1] * T / 2 + a[2] * T**2 / 3 + a[3] * T**3 / 4 + a[4] * T**4 / 5 + a[5] / T
    s = a[0] * math.log(T) + a[1] * T + a[2] * T**2 / 2 + a[3] * T**3 / 3 + a[4] * T**4 / 4 + a[6]
    return cp, h, s


def check_thermo(name):
    comp, lo, hi = THERMO[name]
    for x, y, what in zip(nasa_eval(lo, 1000.0), nasa_eval(hi, 1000.0), ("cp/R", "h/RT", "s/R")):
        if abs(x - y) > 2e-3 * max(1.0, abs(x)):
            raise SystemExit(f"thermo discontinuity at Tmid for {name} in {what}: {x} vs {y}")


def build(name, spec):
    species = spec["species"]
    idx = {s: i for i, s in enumerate(species)}
    sp = []
    for s in species:
        check_thermo(s)
        comp, lo, hi = THERMO[s]
        W = sum(ATOMIC[e] * c for e, c in comp.items())
        sp.append({"name": s, "composition": comp, "W": W,
                   "nasa": {"Tmid": 1000.0, "low": lo, "high": hi}})
    rx = []
    for eq, A, b, Ea, ex in spec["reactions"]:
        lhs, rhs = eq.split("<=>")
        reac, m1 = parse_side(lhs)
        prod, m2 = parse_side(rhs)
        typ = ex.get("type", "elementary")
        if typ == "tb":
            assert m1 and m2, eq
        for side in (reac, prod):
            assert 1 <= len(side) <= 3, eq
            for s in side:
                assert s in idx, (eq, s)
        # element balance
        bal = {}
        for s in reac:
            for e, c in THERMO[s][0].items():
                bal[e] = bal.get(e, 0) + c
        for s in prod:
            for e, c in THERMO[s][0].items():
                bal[e] = bal.get(e, 0) - c
        if any(v != 0 for v in bal.values()):
            raise SystemExit(f"{name}: reaction not element balanced: {eq}")
        r = {"equation": eq, "reactants": reac, "products": prod, "reversible": True,
             "type": {"elementary": "elementary", "tb": "three_body", "lind": "lindemann",
                      "troe": "troe"}[typ],
             "A": A, "b": b, "Ea": Ea}
        if typ in ("tb", "lind", "troe"):
            eff = {s: 1.0 for s in species}
            for s, v in ex.get("eff", {}).items():
                if s in idx:
                    eff[s] = v
            r["efficiencies"] = eff
        if typ in ("lind", "troe"):
            A0, b0, E0 = ex["low"]
            r["low"] = {"A": A0, "b": b0, "Ea": E0}
        if typ == "troe":
            r["troe"] = list(ex["troe"])
        rx.append(r)
    return {"name": name, "provenance": spec["provenance"], "units": {"A": "cm,mol,s", "Ea": "cal/mol"},
            "species": sp, "reactions": rx}


def main():
    # sanity: standard enthalpies of formation [kcal/mol] at 298.15 K
    R_kcal = 1.98720425864083e-3
    for s, dHf in (("H2O", -57.80), ("CO2", -94.05), ("OH", 8.9), ("CH4", -17.9), ("CO", -26.4)):
        comp, lo, hi = THERMO[s]
        h = nasa_eval(lo, 298.15)[1] * R_kcal * 298.15
        if abs(h - dHf) > 0.6:
            raise SystemExit(f"dHf check failed for {s}: {h} vs {dHf}")
    for name, spec in MECHS.items():
        tab = build(name, spec)
        with open(os.path.join(HERE, name + ".json"), "w") as f:
            json.dump(tab, f, indent=1)
        print(f"{name}: K={len(tab['species'])} reactions={len(tab['reactions'])}")


if __name__ == "__main__":
    main()
