"""CPU checks of the C-ABI library: it loads without a GPU, exports every
symbol include/bdfb.h declares, and validates arguments without touching the
device.  No compute calls (there is no GPU here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "bdfb.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2405_01713_b200 import _lib
    from paper_2405_01713_b200 import build as B
    B.build()
    return _lib.lib()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bdfb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding_symbols():
    from paper_2405_01713_b200 import _lib
    assert sorted(_lib.SYMBOLS) == declared_symbols()


def test_library_exports_every_declared_symbol(lib):
    raw = C.CDLL(os.path.join(REPO, "paper_2405_01713_b200", "libbdfb.so"))
    for s in declared_symbols():
        assert hasattr(raw, s), s
    assert lib.bdfb_version().decode().endswith("sm_100a")


def test_argument_validation_without_device(lib):
    from paper_2405_01713_b200 import _lib as L
    h = C.c_void_p()
    atol = np.full(3, 1e-10)
    ap = atol.ctypes.data_as(C.POINTER(C.c_double))
    opt = L.Options()
    lib.bdfb_default_options(C.byref(opt))
    assert (opt.qmax, opt.mode, opt.mxstep) == (5, 0, 10000)
    assert lib.bdfb_create(C.byref(h), 0, 3, 1e-6, ap, C.byref(opt), 0) == -1      # n_cells
    assert lib.bdfb_create(C.byref(h), 10, 0, 1e-6, ap, C.byref(opt), 0) == -1     # n
    assert lib.bdfb_create(C.byref(h), 10, 65, 1e-6, ap, C.byref(opt), 0) == -1    # n > 64
    assert lib.bdfb_create(C.byref(h), 10, 3, 0.0, ap, C.byref(opt), 0) == -1      # rtol
    bad = np.array([1e-10, -1.0, 1e-10])
    assert lib.bdfb_create(C.byref(h), 10, 3, 1e-6, bad.ctypes.data_as(C.POINTER(C.c_double)), C.byref(opt), 0) == -1
    opt.qmax = 6
    assert lib.bdfb_create(C.byref(h), 10, 3, 1e-6, ap, C.byref(opt), 0) == -1
    assert b"qmax" in lib.bdfb_last_error(None)
    # null handles are rejected, not dereferenced
    assert lib.bdfb_set_model(None, 1, None, 0) == -1
    assert lib.bdfb_integrate(None, 0.0, 1.0, None, None, None, 0, None) == -1
    assert lib.bdfb_get_stats(None, None) == -1
    lib.bdfb_destroy(None)


def test_product_package_has_no_oracle_or_cpu_fallback():
    """The product path must not import oracle/ and must fail loudly without libbdfb.so."""
    pkg = os.path.join(REPO, "paper_2405_01713_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).replace("oracle/", ""), f
    from paper_2405_01713_b200 import _lib
    saved = _lib.LIB_PATH, _lib._lib
    try:
        _lib.LIB_PATH, _lib._lib = "/nonexistent/libbdfb.so", None
        with pytest.raises(_lib.LibraryMissing):
            _lib.lib()
    finally:
        _lib.LIB_PATH, _lib._lib = saved
