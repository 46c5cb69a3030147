"""The C-ABI library builds, loads and exports every symbol the header
declares (no compute calls: this runs without a GPU)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1811_09599_b200 import _lib

HEADER = os.path.join(ROOT, "include", "qflex_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(qf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_table():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_library_is_built_for_sm100a():
    import subprocess
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_error_strings_without_gpu():
    lib = _lib.load()
    assert lib.qf_version() >= 100
    # argument validation happens before any device work
    dims = _lib.dims_array([2, 2])
    perm = _lib.perm_array([0, 0])
    st = lib.qf_permute(None, None, 2, dims, perm, 8, None)
    assert st == _lib.QF_ERR_INVALID
    assert b"permutation" in lib.qf_last_error()
    with pytest.raises(ValueError):
        _lib.check(st, "permute")
