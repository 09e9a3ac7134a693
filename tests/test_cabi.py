"""The C-ABI boundary (CPU, no compute): libdpipe.so loads, exports every entry point
include/dpipe.h declares, and the ctypes binding covers exactly that set. The product
path fails loudly when the library is missing (no fallback)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dpipe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dp_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_2405_01248_b200 import _lib

    assert _declared() == sorted(_lib.exported_symbols())


def test_library_exports_every_symbol():
    from paper_2405_01248_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libdpipe.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing
    L = _lib.lib()
    assert L.dp_version() >= 1
    # a size query is pure host code and is safe without a GPU
    assert L.dp_group_norm_workspace(2, 64, 32) > 0


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2405_01248_b200 import _lib

    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.DpipeError):
        _lib.lib()
