"""Build libbdfb.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Steps: (1) codegen: mechanisms/*.json -> csrc/gen/mech_*.cuh; (2) nvcc
-gencode arch=compute_100a,code=sm_100a -lineinfo into
paper_2405_01713_b200/libbdfb.so.  Rebuilds only when a source is newer.
-fmad=false: no implicit contraction, so decision-feeding scalar arithmetic
follows the listing's operation order; fma() is written where intended.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libbdfb.so")
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
UNITS = ["bdfb.cu", "tpc.cu", "split.cu", "split_mf.cu", "erk.cu", "rhs.cu"]
# contraction (a*b + c -> DFMA) only where the parity bar allows it: the generated RHS kernels (R19)
UNIT_FMAD = {}   # measured: -fmad=true for rhs.cu made K_rhs 3% slower (more spills; profiles/r2/history.md)


def sources():
    return (glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
            glob.glob(os.path.join(REPO, "include", "*.h")) + glob.glob(os.path.join(REPO, "mechanisms", "*.json")) +
            [os.path.join(PKG, "codegen", "gen_mech.py"), os.path.join(PKG, "codegen", "gen_tpc.py"), __file__])


def unit_deps(path: str, seen=None) -> set:
    """The file and every quoted #include it reaches (transitively), for per-unit rebuild decisions."""
    seen = set() if seen is None else seen
    path = os.path.normpath(path)
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as f:
        for line in f:
            s = line.strip()
            if s.startswith("#include \""):
                unit_deps(os.path.join(os.path.dirname(path), s.split('"')[1]), seen)
    return seen


def build(force: bool = False, verbose: bool = False) -> str:
    sys.path.insert(0, REPO)
    from paper_2405_01713_b200.codegen import gen_mech, gen_tpc
    gen_mech.main([])
    gen_tpc.main([])
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(s) <= t for s in sources()):
            return LIB
    objs, procs = [], []
    always = [__file__] + glob.glob(os.path.join(REPO, "mechanisms", "*.json"))
    for u in UNITS:
        obj = os.path.join(PKG, "build", u.replace(".cu", ".o"))
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        objs.append(obj)
        deps = list(unit_deps(os.path.join(CSRC, u))) + always
        if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in deps):
            procs.append(None)     # object up to date with every file the unit includes
            continue
        fl = [UNIT_FMAD.get(u, f) if f == "-fmad=false" else f for f in FLAGS]
        procs.append(subprocess.Popen([NVCC] + ARCH + fl + ["-c", "-o", obj, os.path.join(CSRC, u)],
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    info, err = [], None
    info_path = os.path.join(PKG, "ptxas_info.txt")
    old = {}
    if os.path.exists(info_path):   # keep the ptxas report of units that were not recompiled
        for chunk in open(info_path).read().split("==== ")[1:]:
            old[chunk.split("\n", 1)[0]] = "==== " + chunk
    for u, p in zip(UNITS, procs):
        if p is None:
            info.append(old.get(u, f"==== {u}\n(up to date)\n"))
            continue
        out, e = p.communicate()
        info.append(f"==== {u}\n{out}{e}")
        if p.returncode != 0:
            err = f"nvcc failed on {u}:\n" + e[-4000:]
    with open(info_path, "w") as f:
        f.write("".join(info))
    if err:
        raise RuntimeError(err)
    r = subprocess.run([NVCC] + ARCH + ["--shared", "-o", LIB + ".tmp"] + objs + ["-lnccl"], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("".join(info))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
