"""ctypes binding of libqflex_b200.so (the C ABI in include/qflex_b200.h).

PyTorch is used only for device buffers and the current CUDA stream; every
numeric operation on the amplitude path goes through this library.  There
is no CPU fallback: importing works without a GPU (so host-side tooling and
the CPU test-suite run anywhere), but any call that needs the library
raises if the shared object is missing or no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libqflex_b200.so")

QF_OK = 0
QF_ERR_INVALID = -1
QF_ERR_CUDA = -2
QF_ERR_MEMORY = -3
QF_ERR_UNSUPPORTED = -4

GEMM_AUTO, GEMM_FFMA, GEMM_TC3 = 0, 1, 2
GATHER_ROWS_UNIT = 0x100  # or'ed into qf_cgemm_c64_gather's mode: roff[r] = roff[0] + r
BOFF_EVEN = 0x200         # or'ed into qf_cgemm_c64_gather_boff's mode: entry bases even
BBOFF_EVEN = 0x400        # or'ed into qf_cgemm_c64_ex's mode: B entry bases even
C_TRANS = 0x800           # or'ed into qf_cgemm_c64_ex's mode: C stored transposed per entry
OP_N, OP_T = 0, 1

# every exported symbol declared in include/qflex_b200.h
EXPORTS = (
    "qf_last_error", "qf_version", "qf_device_info", "qf_permute", "qf_permute_c64",
    "qf_gather_axis", "qf_fix_axis", "qf_cgemm_c64", "qf_cgemm_c64_gather", "qf_zgemm_c128",
    "qf_bit_offsets", "qf_gather_rows", "qf_cgemm_c64_gather_boff", "qf_cgemm_c64_ex",
    "qf_cgemm_c64_ex2", "qf_cgemm_c64_tview", "qf_cgemm_c64_view2",
    "qf_cgemm_c64_view", "qf_sv_basis", "qf_sv_apply", "qf_sv_gather",
    "qf_accumulate",
    "qf_fill_zero", "qf_tc3_set_variant", "qf_last_kernel",
    "qf_small_engine", "qf_rowmma", "qf_cgemm_c64_rowblocks",
    "qf_workspace_reserve", "qf_workspace_release", "qf_launch_count",
    "qf_nccl_available", "qf_nccl_unique_id", "qf_nccl_init", "qf_nccl_destroy",
    "qf_allreduce_c64", "qf_axpy_c64", "qf_dot_c64", "qf_affine_offsets", "qf_fill_value",
)


class LibraryMissingError(RuntimeError):
    """The CUDA library is not built (or not loadable) on this machine."""


class MemoryBudgetError(RuntimeError):
    """Executing (or estimating) a plan would exceed the memory budget
    (mirrors rqcsim.contraction_plan.MemoryBudgetError, rq/contraction_plan.py:56)."""


_lib = None
_lock = threading.Lock()

_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def _declare(lib):
    lib.qf_last_error.restype = ctypes.c_char_p
    lib.qf_last_error.argtypes = []
    lib.qf_version.restype = ctypes.c_int
    lib.qf_device_info.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    lib.qf_permute.argtypes = [_c_void_p, _c_void_p, ctypes.c_int, ctypes.POINTER(_i64),
                               ctypes.POINTER(_i32), ctypes.c_int, _c_void_p]
    lib.qf_permute_c64.argtypes = [_c_void_p, _c_void_p, ctypes.c_int, ctypes.POINTER(_i64),
                                   ctypes.POINTER(_i32), _c_void_p]
    lib.qf_gather_axis.argtypes = [_c_void_p, _c_void_p, _i64, _i64, _i64, _c_void_p, _i64,
                                   ctypes.c_int, _c_void_p]
    lib.qf_fix_axis.argtypes = [_c_void_p, _c_void_p, _i64, _i64, _i64, _i64, ctypes.c_int,
                                _c_void_p]
    lib.qf_cgemm_c64.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64,
                                 _c_void_p, _i64, _i64, ctypes.c_int,
                                 _c_void_p, _i64, _i64, ctypes.c_int,
                                 _c_void_p, _i64, _i64,
                                 ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                 _c_void_p]
    lib.qf_cgemm_c64_gather.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64,
                                        _c_void_p, _i64, _c_void_p, _c_void_p,
                                        _c_void_p, _i64, _i64, ctypes.c_int,
                                        _c_void_p, _i64, _i64,
                                        ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                        ctypes.c_float, _c_void_p]
    lib.qf_cgemm_c64_gather_boff.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64,
                                             _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                                             _c_void_p, _i64, _i64, ctypes.c_int,
                                             _c_void_p, _i64, _i64,
                                             ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                             ctypes.c_float, _c_void_p]
    lib.qf_cgemm_c64_ex.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64,
                                    _c_void_p, _i64, _i64, ctypes.c_int, _c_void_p, _c_void_p,
                                    _c_void_p, _c_void_p, _i64, _i64, ctypes.c_int, _c_void_p,
                                    _c_void_p, _i64, _i64,
                                    ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                    ctypes.c_float, _c_void_p]
    lib.qf_cgemm_c64_ex2.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64,
                                     _c_void_p, _i64, _i64, ctypes.c_int, _c_void_p, _i64, _c_void_p,
                                     _c_void_p, _c_void_p, _i64, _i64, ctypes.c_int, _c_void_p,
                                     _i64, _c_void_p, _i64, _i64,
                                     ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                     ctypes.c_float, _c_void_p]
    lib.qf_cgemm_c64_tview.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64, _c_void_p, _i64,
                                       _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                                       _c_void_p, _i64, _i64, ctypes.c_int, _c_void_p, _i64,
                                       _c_void_p, _i64, _i64,
                                       ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                       ctypes.c_float, _c_void_p]
    lib.qf_cgemm_c64_view2.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64, _c_void_p, _i64,
                                       _c_void_p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                                       _c_void_p, _i64, _i64, ctypes.c_int, _c_void_p, _i64,
                                       _c_void_p, _i64, _i64, _i64, _i64,
                                       ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                       ctypes.c_float, _c_void_p]
    lib.qf_cgemm_c64_view.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64, _c_void_p, _i64,
                                      _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                                      _c_void_p, _i64, _i64, ctypes.c_int, _c_void_p, _i64,
                                      _c_void_p, _i64, _i64,
                                      ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                      ctypes.c_float, _c_void_p]
    lib.qf_sv_basis.argtypes = [_c_void_p, ctypes.c_int, _i64, _c_void_p]
    lib.qf_sv_apply.argtypes = [_c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i32),
                                ctypes.c_int, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                ctypes.POINTER(ctypes.c_double), _c_void_p]
    lib.qf_sv_gather.argtypes = [_c_void_p, _c_void_p, _i64, _c_void_p, _c_void_p]
    lib.qf_bit_offsets.argtypes = [_c_void_p, _i64, ctypes.c_int, ctypes.POINTER(_i32),
                                   ctypes.POINTER(_i64), _i64, _c_void_p, _c_void_p]
    lib.qf_gather_rows.argtypes = [_c_void_p, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                   ctypes.c_int, _c_void_p]
    lib.qf_zgemm_c128.argtypes = [_i64, _i64, _i64, _i64,
                                  _c_void_p, _i64, _i64, ctypes.c_int,
                                  _c_void_p, _i64, _i64, ctypes.c_int,
                                  _c_void_p, _i64, _i64,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, _c_void_p]
    lib.qf_accumulate.argtypes = [_c_void_p, _c_void_p, _i64, ctypes.c_int, _c_void_p]
    lib.qf_fill_zero.argtypes = [_c_void_p, _i64, _c_void_p]
    lib.qf_tc3_set_variant.argtypes = [ctypes.c_int]
    lib.qf_small_engine.argtypes = [ctypes.c_int]
    lib.qf_rowmma.argtypes = [ctypes.c_int]
    lib.qf_cgemm_c64_rowblocks.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64, _c_void_p, _i64,
                                           _i64, _i64, _i64, _c_void_p, _i64, _i64, ctypes.c_int,
                                           _c_void_p, _i64, _i64, ctypes.c_float, ctypes.c_float,
                                           ctypes.c_float, ctypes.c_float, _c_void_p]
    lib.qf_last_kernel.restype = ctypes.c_char_p
    lib.qf_last_kernel.argtypes = []
    lib.qf_workspace_reserve.argtypes = [_i64, _c_void_p]
    lib.qf_workspace_release.argtypes = []
    lib.qf_nccl_available.argtypes = []
    lib.qf_nccl_unique_id.argtypes = [_c_void_p, _i64]
    lib.qf_nccl_init.argtypes = [_c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_int)]
    lib.qf_nccl_destroy.argtypes = [ctypes.c_int]
    lib.qf_allreduce_c64.argtypes = [ctypes.c_int, _c_void_p, _i64, _c_void_p]
    lib.qf_axpy_c64.argtypes = [_i64, ctypes.c_float, ctypes.c_float, _c_void_p, _c_void_p,
                                _c_void_p]
    lib.qf_dot_c64.argtypes = [_i64, _i64, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _c_void_p]
    lib.qf_affine_offsets.argtypes = [_c_void_p, _i64, _i64, _i64, _c_void_p, _i64, _c_void_p]
    lib.qf_fill_value.argtypes = [_c_void_p, _i64, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                  _c_void_p]
    lib.qf_launch_count.argtypes = [ctypes.c_int]
    lib.qf_launch_count.restype = _i64
    for name in EXPORTS:
        if name not in ("qf_last_error", "qf_launch_count", "qf_last_kernel"):
            getattr(lib, name).restype = ctypes.c_int
    return lib


def load(path: Optional[str] = None):
    """Load (once) and return the ctypes handle; raises LibraryMissingError."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise LibraryMissingError(
                f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = _declare(ctypes.CDLL(p))
        except OSError as exc:  # pragma: no cover - depends on the box
            raise LibraryMissingError(f"cannot load {p}: {exc}") from None
        if path is None:
            _lib = lib
        return lib


def check(status: int, what: str = "qflex"):
    if status == QF_OK:
        return
    msg = load().qf_last_error().decode(errors="replace")
    if status == QF_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    if status == QF_ERR_MEMORY:
        raise MemoryBudgetError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({status}): {msg}")


def dims_array(dims: Sequence[int]):
    return (_i64 * max(1, len(dims)))(*[int(d) for d in dims])


def perm_array(perm: Sequence[int]):
    return (_i32 * max(1, len(perm)))(*[int(p) for p in perm])


def launch_count(reset: bool = False) -> int:
    return int(load().qf_launch_count(1 if reset else 0))


# -- multi-GPU slice collective (qf_nccl_* / qf_allreduce_c64) ----------------

NCCL_UID_BYTES = 128


def _current_stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 of a group draws it; the host
    broadcasts the bytes to the other ranks)."""
    buf = ctypes.create_string_buffer(NCCL_UID_BYTES)
    check(load().qf_nccl_unique_id(buf, NCCL_UID_BYTES), "nccl_unique_id")
    return buf.raw


def nccl_init(uid: bytes, nranks: int, rank: int, device: int) -> int:
    """Join the communicator named by `uid` as `rank` of `nranks` on
    `device`; returns the library handle (collective over all ranks)."""
    if len(uid) != NCCL_UID_BYTES:
        raise ValueError(f"NCCL unique id must be {NCCL_UID_BYTES} bytes, got {len(uid)}")
    h = ctypes.c_int(-1)
    buf = ctypes.create_string_buffer(uid, NCCL_UID_BYTES)
    check(load().qf_nccl_init(buf, int(nranks), int(rank), int(device), ctypes.byref(h)),
          "nccl_init")
    return int(h.value)


def nccl_destroy(handle: int):
    check(load().qf_nccl_destroy(int(handle)), "nccl_destroy")


def allreduce_c64(handle: int, buf, count: int):
    """In-place sum of `count` complex64 values of a device buffer over the
    communicator, on the current CUDA stream."""
    check(load().qf_allreduce_c64(int(handle), ctypes.c_void_p(buf.data_ptr()), int(count),
                                  _current_stream()), "allreduce_c64")


def axpy_c64(x, y, alpha: complex = 1.0, n: Optional[int] = None):
    """y[:n] += alpha * x[:n] on the device (complex64)."""
    n = int(x.numel()) if n is None else int(n)
    a = complex(alpha)
    check(load().qf_axpy_c64(n, a.real, a.imag, ctypes.c_void_p(x.data_ptr()),
                             ctypes.c_void_p(y.data_ptr()), _current_stream()), "axpy_c64")


def dot_c64(x, y, out, batch: int, n: int, stride_x: Optional[int] = None,
            stride_y: Optional[int] = None):
    """out[b] = sum_i x[b, i] * y[b, i] on the device (complex64)."""
    sx = n if stride_x is None else int(stride_x)
    sy = n if stride_y is None else int(stride_y)
    check(load().qf_dot_c64(int(batch), int(n), ctypes.c_void_p(x.data_ptr()), sx,
                            ctypes.c_void_p(y.data_ptr()), sy, ctypes.c_void_p(out.data_ptr()),
                            _current_stream()), "dot_c64")


def last_kernel() -> str:
    """Name of the kernel family the library launched last on this thread."""
    return load().qf_last_kernel().decode()
