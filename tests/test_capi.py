"""The C-ABI library loads and exports every symbol include/blfls/blfls.h
declares (no compute calls without a GPU), and the host mirror validates like
the reference before touching the device."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "blfls" / "blfls.h").read_text()
    return sorted(set(re.findall(r"\b(blfls_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1812_07122_b200 import build
    path = build.build()
    return ctypes.CDLL(str(path))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for s in ("blfls_plan_create", "blfls_run", "blfls_solve", "blfls_filter_gradients",
              "blfls_rfft2", "blfls_irfft2", "blfls_last_error"):
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_lists_all_exports():
    from paper_1812_07122_b200 import _capi
    assert sorted(_capi.EXPORTS) == header_symbols()


def test_abi_version_and_strings(lib):
    lib.blfls_abi_version.restype = ctypes.c_int
    lib.blfls_version.restype = ctypes.c_char_p
    assert lib.blfls_abi_version() == 3
    assert b"sm_100a" in lib.blfls_version()


def test_plan_create_validation_without_gpu(lib):
    """Parameter validation mirrors bilateral.cpp:12-16 / solver.cpp:15-21 and
    happens before any device call; without a device the call fails loudly."""
    from paper_1812_07122_b200 import _capi
    L = _capi.lib()
    h = ctypes.c_void_p()
    bad = [
        _capi.Params(1, 16, 1, 0, 3, 1.0, 0.1, 1.0, 1, 0),     # height < 2
        _capi.Params(16, 16, 2, 0, 3, 1.0, 0.1, 1.0, 1, 0),    # channels
        _capi.Params(16, 16, 1, 2, 3, 1.0, 0.1, 1.0, 1, 0),    # guide channels
        _capi.Params(16, 16, 1, 0, 3, 0.0, 0.1, 1.0, 1, 0),    # sigma_s
        _capi.Params(16, 16, 1, 0, 3, 1.0, -0.1, 1.0, 1, 0),   # sigma_r
        _capi.Params(16, 16, 1, 0, 3, 1.0, 0.1, -1.0, 1, 0),   # lambda
        _capi.Params(16, 16, 1, 0, 3, 1.0, 0.1, float("nan"), 1, 0),
        _capi.Params(16, 16, 1, 0, 3, 1.0, 0.1, 1.0, 1, 0, -1),    # pad < 0
    ]
    for p in bad:
        assert L.blfls_plan_create(ctypes.byref(p), ctypes.byref(h)) == _capi.BLFLS_EINVAL
        assert L.blfls_last_error()
    big = _capi.Params(16, 16, 1, 0, 200, 1.0, 0.1, 1.0, 1, 0)
    assert L.blfls_plan_create(ctypes.byref(big), ctypes.byref(h)) == _capi.BLFLS_EUNSUPPORTED
    import torch
    if not torch.cuda.is_available():
        ok = _capi.Params(16, 16, 1, 0, 3, 1.0, 0.1, 1.0, 1, 0)
        assert L.blfls_plan_create(ctypes.byref(ok), ctypes.byref(h)) == _capi.BLFLS_ECUDA


def test_host_mirror_rejects_bad_shapes():
    import paper_1812_07122_b200 as P
    with pytest.raises(P.InvalidArgument):
        P.blf_ls(np.zeros((2, 8, 8), np.float32), lam=1.0, sigma_s=1.0, sigma_r=0.1)
    with pytest.raises(P.InvalidArgument):
        P.blf_ls(np.zeros((8, 8), np.float32), np.zeros((9, 8), np.float32), lam=1.0,
                 sigma_s=1.0, sigma_r=0.1)
    with pytest.raises(P.InvalidArgument):
        P.blf_ls(np.zeros((8, 8), np.float32), lam=1.0, sigma_s=1.0, sigma_r=0.1, pad=-1)


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = ROOT / "paper_1812_07122_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        for bad in ("from oracle", "import oracle", "liboracle", "libepls_ref", "orc_"):
            assert bad not in text, (f, bad)


def test_multi_create_validation_without_gpu():
    """blfls_multi_create validates before touching a device."""
    from paper_1812_07122_b200 import _capi
    L = _capi.lib()
    h = ctypes.c_void_p()
    ok = _capi.Params(64, 64, 1, 0, 3, 1.0, 0.1, 1.0, 2, 0, 0, 0, 0)
    devs = (ctypes.c_int * 2)(0, 0)
    assert L.blfls_multi_create(ctypes.byref(ok), devs, 0, 0, ctypes.byref(h)) == _capi.BLFLS_EINVAL
    assert L.blfls_multi_create(ctypes.byref(ok), devs, 9, 0, ctypes.byref(h)) == _capi.BLFLS_EINVAL
    assert L.blfls_multi_create(ctypes.byref(ok), devs, 2, 7, ctypes.byref(h)) == _capi.BLFLS_EINVAL
    # band mode: one image only, brute force, pad 0
    assert L.blfls_multi_create(ctypes.byref(ok), devs, 2, _capi.MULTI_BAND, ctypes.byref(h)) == _capi.BLFLS_EINVAL
    padded = _capi.Params(64, 64, 1, 0, 3, 1.0, 0.1, 1.0, 1, 0, 16, 0, 0)
    assert L.blfls_multi_create(ctypes.byref(padded), devs, 2, _capi.MULTI_BAND,
                                ctypes.byref(h)) == _capi.BLFLS_EUNSUPPORTED
    assert L.blfls_multi_run(None, None, None, 1, 1, None, 1) == _capi.BLFLS_EINVAL
