"""The C-ABI library (libqbg.so) loads and exports every symbol declared in include/qbg.h;
without a GPU, device calls fail loudly (no CPU fallback).  CPU only."""
import ctypes
import os
import re

import pytest

from conftest import ROOT, cuda_available
from paper_1912_10877_b200 import _capi, errors


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "qbg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qbg_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = _capi.lib()
    syms = declared_symbols()
    assert len(syms) > 50
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_capi.QbgOp) == 192
    assert ctypes.sizeof(_capi.QbgPauliTerm) == 32


def test_host_only_entry_points():
    lib = _capi.lib()
    assert lib.qbg_version().startswith(b"qbg")
    h = ctypes.c_void_p()
    _capi.check(lib.qbg_rng_create(42, ctypes.byref(h)))
    u = lib.qbg_rng_uniform(h)
    assert 0.0 <= u < 1.0
    lib.qbg_rng_destroy(h)
    old = lib.qbg_get_qubit_cap()
    _capi.check(lib.qbg_set_qubit_cap(36))
    assert lib.qbg_get_qubit_cap() == 36
    _capi.check(lib.qbg_set_qubit_cap(old))
    with pytest.raises(errors.ValidationError):
        _capi.check(lib.qbg_set_qubit_cap(0))


def test_host_rng_matches_reference_stream(golden):
    from paper_1912_10877_b200.register import Rng
    g = golden("rng.npz")
    r = Rng(42)
    assert [r.uniform() for _ in range(64)] == g["uniform"].tolist()


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure mode")
def test_device_calls_fail_loudly_without_gpu():
    from paper_1912_10877_b200 import zero_state
    with pytest.raises(errors.CudaError):
        zero_state(3)
