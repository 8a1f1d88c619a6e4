"""The C-ABI library loads and exports every symbol include/alefsi_b200.h
declares (CPU only: no compute calls that need a device)."""

import os
import re

import numpy as np

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "alefsi_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(alefsi_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1904_02401_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if getattr(lib, s, None) is None]
    assert not missing, missing
    # and the Python binding declares exactly the header's functions
    assert sorted(_lib.SIGNATURES) == syms


def test_abi_version_and_error_string():
    from paper_1904_02401_b200 import _lib
    lib = _lib.load()
    assert lib.alefsi_abi_version() == 1
    bad = np.zeros(3, dtype=np.int64)
    try:
        _lib.call("alefsi_color_patches", 1, np.array([0, 1], dtype=np.int64),
                  np.array([5], dtype=np.int64), np.array([3], dtype=np.int64), 2, bad, bad)
    except _lib.NativeError as exc:
        assert exc.code == 1 and "out of range" in str(exc)
    else:
        raise AssertionError("expected an argument error")


def test_gmres_has_no_cpu_path():
    import pytest
    import scipy.sparse as sp
    from paper_1904_02401_b200 import linsolve
    with pytest.raises(TypeError):
        linsolve.gmres(sp.identity(4), np.ones(4), preconditioner=None)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_1904_02401_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "absent.so"))
    try:
        _lib.load()
    except ImportError as exc:
        assert "no CPU fallback" in str(exc)
    else:
        raise AssertionError("expected ImportError")
