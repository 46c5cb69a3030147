"""ctypes loader of oracle/permute_ref.c -- TEST INFRASTRUCTURE ONLY.

The bit-exact CPU permutation checker for config 3 (a C restatement of
rq/tensor_core.py:271-273, see permute_ref.c).  Imported only by tests/ and
bench.py's checker legs; the product package never loads it."""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "permute_ref.c")
LIB = os.path.join(HERE, "lib", "libpermute_ref.so")
_lib = None


def build() -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", SRC, "-o", LIB])
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
            build()
        lib = ctypes.CDLL(LIB)
        lib.permute_ref.restype = ctypes.c_int
        lib.permute_ref.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32),
                                    ctypes.c_int]
        _lib = lib
    return _lib


def permute(src: np.ndarray, dims: Sequence[int], perm: Sequence[int],
            out: np.ndarray = None) -> np.ndarray:
    """ascontiguousarray(transpose(src.reshape(dims), perm)).reshape(-1), bit-exact."""
    src = np.ascontiguousarray(src).reshape(-1)
    if out is None:
        out = np.empty_like(src)
    r = len(dims)
    d = (ctypes.c_int64 * max(r, 1))(*[int(x) for x in dims])
    p = (ctypes.c_int32 * max(r, 1))(*[int(x) for x in perm])
    st = load().permute_ref(src.ctypes.data, out.ctypes.data, r, d, p, src.itemsize)
    if st != 0:
        raise ValueError(f"bad permutation {list(perm)} of dims {list(dims)}")
    return out
