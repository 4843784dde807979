"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every entry point
include/hdgb200.h declares, and refuses to run without a CUDA device (no CPU fallback)."""
import ctypes
import re
from pathlib import Path

import pytest

import paper_2512_13619_b200 as hdg
from paper_2512_13619_b200 import hdg as H

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "hdgb200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hdgb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(hdg.library_path()))
    names = declared_symbols()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_mirror_binds_every_declared_symbol():
    assert set(H.exported_symbols()) == set(declared_symbols())


def test_host_only_entry_points_work_without_gpu():
    # leja_order is pure host code behind the ABI (preconditioner.cpp:207-244)
    out = hdg.leja_order([1.0, 2.0, 3.0, 4.0])
    assert out[0] == 4.0 and out[1] == 1.0
    out = hdg.leja_order([1 + 2j, 1 - 2j, 5.0])
    assert out[0] == 5.0 and out[1] == 1 + 2j and out[2] == 1 - 2j


def test_no_cpu_fallback(monkeypatch):
    from conftest import _has_gpu
    if _has_gpu():
        pytest.skip("a CUDA device is present")
    with pytest.raises(hdg.CudaError):
        hdg.Context(0)


def test_reference_generator_restated():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref missing")
    import numpy as np
    assert np.array_equal(hdg.random_vector(50, 12345, 0.5), ref.random_vector(50, 12345, 0.5))
