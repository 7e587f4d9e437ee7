"""paper_2405_01713_b200 -- batched stiff-ODE integration (CVODE-style BDF) on B200.

Thin Python binding over the C ABI of libbdfb.so (include/bdfb.h): argument
marshalling only.  Every step of the hot path runs in the CUDA kernels of
csrc/; PyTorch provides device memory, streams and process groups.  There is
no CPU fallback: a missing or unloadable libbdfb.so raises.

    import torch, paper_2405_01713_b200 as bdfb
    b = bdfb.Batch(n_cells=N, n=22, rtol=1e-6, atol=1e-10)
    b.set_model("drm19")
    b.integrate(0.0, 1e-5, y, f_ext=F, aux=rho)       # y: cuda fp64 [n, N] (YC)
    print(b.stats())
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

MODE_PER_CELL, MODE_GLOBAL_NORM = L.MODE_PER_CELL, L.MODE_GLOBAL_NORM

__all__ = ["Batch", "MODE_PER_CELL", "MODE_GLOBAL_NORM", "MODELS", "eval_rhs", "eval_jac", "lu_factor_solve", "version", "library_path"]

MODELS = {"linear": (L.MODEL_LINEAR, 1), "robertson": (L.MODEL_ROBERTSON, 3), "nyx_kwh": (L.MODEL_NYX_KWH, 1),
          "h2": (L.MODEL_MECH_H2, 10), "drm19": (L.MODEL_MECH_DRM19, 22), "gri53": (L.MODEL_MECH_GRI53, 54)}
STATUS = {0: "OK", 1: "TOO_MUCH_WORK", 2: "ERR_FAILURE", 3: "CONV_FAILURE", 4: "RHS_FAIL", 5: "NONFINITE_INPUT"}
CELL_STAT_FIELDS = ["status", "nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn", "q_last", "h_last", "t_reached"]


def torch_empty_like(t):
    import torch
    return torch.empty_like(t)


def library_path():
    return L.LIB_PATH


def version():
    return L.lib().bdfb_version().decode()


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if t.dtype.itemsize != 8 and t.dtype.is_floating_point:
            raise TypeError("fp64 tensors required")
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(t.ctypes.data)
    raise TypeError(f"unsupported buffer {type(t)}")


def _dev(t, batch, numel, name, dtype="f64", optional=True):
    """Validated device pointer for the C ABI (which takes no lengths): a contiguous CUDA tensor on the
    batch's device with the expected dtype and element count; None passes through when optional."""
    import torch
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.device.index != batch.device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the batch on cuda:{batch.device}")
    want = {"f64": torch.float64, "i32": torch.int32}[dtype]
    if t.dtype != want:
        raise TypeError(f"{name} must be {want}, got {t.dtype}")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return C.c_void_p(t.data_ptr())


def _host(a, numel, name, optional=True):
    """Validated host buffer (numpy float64 or CPU tensor) of numel elements."""
    if a is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    if hasattr(a, "data_ptr"):
        import torch
        if a.is_cuda or a.dtype != torch.float64 or a.numel() != numel or not a.is_contiguous():
            raise ValueError(f"{name} must be a contiguous CPU float64 tensor of {numel} elements")
        return C.c_void_p(a.data_ptr())
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.size != numel or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{name} must be a C-contiguous float64 array of {numel} elements")
    return C.c_void_p(a.ctypes.data)


def _stream(stream, device=None):
    """The caller's stream; default: torch's current stream on `device` (the batch's device)."""
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _check(rc, handle=None):
    if rc < 0:
        msg = L.lib().bdfb_last_error(handle).decode()
        raise RuntimeError(f"libbdfb error {rc}: {msg}")
    return rc


class Batch:
    """A batch of n_cells independent ODE systems of size n (bdfb_create)."""

    def __init__(self, n_cells, n, rtol, atol, qmax=5, mxstep=10000, h0=0.0, hmin=0.0, hmax=0.0, device=0,
                 mode=L.MODE_PER_CELL):
        self._L = L.lib()
        atol = np.ascontiguousarray(np.broadcast_to(np.asarray(atol, dtype=np.float64), (n,)))
        opt = L.Options(qmax, mode, mxstep, h0, hmin, hmax)
        h = C.c_void_p()
        _check(self._L.bdfb_create(C.byref(h), int(n_cells), int(n), float(rtol),
                                   atol.ctypes.data_as(C.POINTER(C.c_double)), C.byref(opt), int(device)))
        self.h = h
        self.n_cells, self.n, self.rtol, self.atol, self.device = int(n_cells), int(n), float(rtol), atol, device
        self._cell_stats = None
        self.model = None

    def set_model(self, model, params=None):
        mid, n = MODELS[model]
        buf, size = None, 0
        if params is not None:
            if model == "nyx_kwh":
                p = L.KwhParams(params["z"], params["X"], params["Y"], params["gamma_ad"],
                                (C.c_double * 3)(*params["gph"]), (C.c_double * 3)(*params["eph"]))
            elif model == "robertson":
                p = (C.c_double * 3)(*params)
            elif model == "linear":
                p = C.c_double(float(params))
            else:
                raise ValueError("mechanism models take no parameters")
            buf, size = C.cast(C.pointer(p), C.c_void_p), C.sizeof(p)
            self._params_keep = p
        _check(self._L.bdfb_set_model(self.h, mid, buf, size), self.h)
        self.model = model

    def set_kernel(self, kernel):
        """Per-cell kernel for the mechanism models: "split" (= "auto", default), "thread" or "group" (bdfb_set_kernel)."""
        kid = {"auto": L.KERNEL_AUTO, "thread": L.KERNEL_THREAD, "group": L.KERNEL_GROUP,
               "split": L.KERNEL_SPLIT}[kernel]
        _check(self._L.bdfb_set_kernel(self.h, kid), self.h)

    def set_jacobian(self, mode):
        """"analytic" (default) or "dq": CVODE's difference-quotient dense Jacobian (bdfb_set_jacobian)."""
        _check(self._L.bdfb_set_jacobian(self.h, {"analytic": 0, "dq": 1}[mode]), self.h)

    def set_method(self, method):
        """"bdf" (default) or "erk4": the explicit adaptive ERK of P:415-426 (bdfb_set_method)."""
        _check(self._L.bdfb_set_method(self.h, {"bdf": 0, "erk4": 1}[method]), self.h)

    def set_linear_solver(self, ls, maxl=0):
        """"dense" (default), "diag" (CVDiag) or "gmres" (inexact Newton-Krylov; maxl
        Krylov iterations, 0 = 5) for the Newton iteration (bdfb_set_linear_solver)."""
        _check(self._L.bdfb_set_linear_solver(self.h, {"dense": 0, "diag": 1, "gmres": 2}[ls], int(maxl)), self.h)

    @property
    def wrms_group(self):
        """Lane-group size of the WRMS summation order (reading R15) the selected kernel uses."""
        return int(self._L.bdfb_wrms_group(self.h))

    def set_comm(self, unique_id: bytes, nranks: int, rank: int, ncells_total: int):
        """Global-norm mode across ranks: NCCL communicator from a 128-byte ncclUniqueId
        (created on rank 0, broadcast by the caller, e.g. with torch.distributed)."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(self._L.bdfb_set_comm(self.h, C.cast(buf, C.c_void_p), int(nranks), int(rank), int(ncells_total)),
               self.h)

    def attach_cell_stats(self, device="cuda"):
        """Allocate per-cell statistics tensors that each integrate fills; returns the dict."""
        import torch
        dev = torch.device(device, self.device) if isinstance(device, str) else device
        d = {}
        for f in CELL_STAT_FIELDS:
            dt = torch.float64 if f in ("h_last", "t_reached") else torch.int32
            d[f] = torch.zeros(self.n_cells, dtype=dt, device=dev)
        cs = L.CellStats(*[C.c_void_p(d[f].data_ptr()) for f in CELL_STAT_FIELDS])
        _check(self._L.bdfb_set_cell_stats(self.h, C.byref(cs)), self.h)
        self._cell_stats = d
        return d

    def detach_cell_stats(self):
        _check(self._L.bdfb_set_cell_stats(self.h, None), self.h)
        self._cell_stats = None

    @property
    def cell_stats(self):
        return self._cell_stats

    def integrate(self, t0, tf, y, f_ext=None, aux=None, layout="YC", stream=None):
        """Advance every cell from t0 to tf in place (y: device fp64, [n, N] for YC or [N, n] for CY)."""
        lay = L.LAYOUT_YC if layout == "YC" else L.LAYOUT_CY
        nn = self.n * self.n_cells
        _check(self._L.bdfb_integrate(self.h, float(t0), float(tf), _dev(y, self, nn, "y", optional=False),
                                      _dev(f_ext, self, nn, "f_ext"), _dev(aux, self, self.n_cells, "aux"), lay,
                                      _stream(stream, self.device)), self.h)

    def integrate_host(self, t0, tf, y, f_ext=None, aux=None, layout="YC", stream=None):
        """End-to-end: host (preferably pinned) buffers in, y copied back; synchronous."""
        lay = L.LAYOUT_YC if layout == "YC" else L.LAYOUT_CY
        nn = self.n * self.n_cells
        _check(self._L.bdfb_integrate_host(self.h, float(t0), float(tf), _host(y, nn, "y", optional=False),
                                           _host(f_ext, nn, "f_ext"), _host(aux, self.n_cells, "aux"), lay,
                                           _stream(stream, self.device)), self.h)

    def stats(self):
        s = L.Stats()
        _check(self._L.bdfb_get_stats(self.h, C.byref(s)), self.h)
        return {f: int(getattr(s, f)) for f, _ in L.Stats._fields_}

    def last_kernel_ms(self):
        return float(self._L.bdfb_last_kernel_ms(self.h))

    def minmax(self, y, layout="YC", stream=None):
        """Per-component min and max of y over the handle's cells (bdfb_minmax); device tensors [n]."""
        import torch
        lo = torch.empty(self.n, dtype=torch.float64, device=y.device)
        hi = torch.empty_like(lo)
        lay = L.LAYOUT_YC if layout == "YC" else L.LAYOUT_CY
        _check(self._L.bdfb_minmax(self.h, _dev(y, self, self.n * self.n_cells, "y", optional=False), lay, _ptr(lo),
                                   _ptr(hi), _stream(stream, self.device)), self.h)
        return lo, hi

    def set_typical_atol(self, y, eta=1e-10, floor=1e-30, layout="YC", group=None, stream=None):
        """Eq. 7 typical-value absolute tolerances from the current field y: the min/max of
        every component over all cells -- of all ranks of `group` when given (torch.distributed MIN/MAX
        reductions of n doubles) -- then atol_i = max(eta (min_i + max_i)/2, floor) on the device.
        Returns the typical values (device tensor [n])."""
        from . import parallel
        lo, hi = self.minmax(y, layout, stream)
        lo, hi = parallel.allreduce_minmax(lo, hi, group)
        tv = torch_empty_like(lo)
        _check(self._L.bdfb_set_atol_typical(self.h, _ptr(lo), _ptr(hi), float(eta), float(floor), _ptr(tv),
                                             _stream(stream)), self.h)
        return tv

    def phase_ms(self):
        """SPLIT kernel: device ms per phase of the last integrate (bdfb_phase_ms), else {}."""
        buf = (C.c_double * 8)()
        n = int(self._L.bdfb_phase_ms(self.h, buf, 8))
        return dict(zip(["ctl", "jac", "lu", "rhs"], list(buf)[:n]))

    def last_launch_count(self):
        return int(self._L.bdfb_last_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self._L.bdfb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def eval_rhs(batch, y, f_ext=None, aux=None, t=0.0, stream=None):
    """f = R(t, y) + F for every cell with the integrator's device RHS (YC layout)."""
    import torch
    nn = batch.n * batch.n_cells
    yp = _dev(y, batch, nn, "y", optional=False)
    f = torch.empty_like(y)
    st = torch.empty(batch.n_cells, dtype=torch.int32, device=y.device)
    _check(batch._L.bdfb_eval_rhs(batch.h, float(t), yp, _dev(f_ext, batch, nn, "f_ext"),
                                  _dev(aux, batch, batch.n_cells, "aux"), _ptr(f), _ptr(st),
                                  _stream(stream, batch.device)), batch.h)
    return f, st


def eval_jac(batch, y, aux=None, t=0.0, stream=None):
    """J[i, j, c] = dR_i/dy_j of every cell with the integrator's device Jacobian."""
    import torch
    yp = _dev(y, batch, batch.n * batch.n_cells, "y", optional=False)
    J = torch.empty((batch.n, batch.n, batch.n_cells), dtype=torch.float64, device=y.device)
    _check(batch._L.bdfb_eval_jac(batch.h, float(t), yp, _dev(aux, batch, batch.n_cells, "aux"), _ptr(J),
                                  _stream(stream, batch.device)), batch.h)
    return J


def lu_factor_solve(M, b, stream=None, routine="tpc"):
    """Batched LU with partial pivoting + solve: M [n, n, N], b [n, N] (cuda fp64).
    Returns (LU, piv, x, info) with LAPACK getrf/getrs conventions.
    routine: "tpc" (bdfb_lu_factor_solve: the thread-per-cell / small-model routine) or "split"
    (bdfb_split_lu_factor_solve: the default SPLIT integrator's oct_factor + Newton-solve substitutions)."""
    import torch
    n, N = b.shape
    LU = M.clone().contiguous()
    x = b.clone().contiguous()
    piv = torch.zeros((n, N), dtype=torch.int32, device=b.device)
    info = torch.zeros(N, dtype=torch.int32, device=b.device)
    fn = L.lib().bdfb_split_lu_factor_solve if routine == "split" else L.lib().bdfb_lu_factor_solve
    _check(fn(int(n), int(N), _ptr(LU), _ptr(piv), _ptr(x), _ptr(info),
                                        _stream(stream)))
    return LU, piv, x, info
