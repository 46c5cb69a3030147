"""Device tensors, index permutation and pairwise contraction on the B200.

Drop-in for the hot-path layer of `rqcsim.tensor_core` (rq/tensor_core.py):

  Tensor(labels, array)            rq/tensor_core.py:338-388  (device-resident here)
  contract(a, b)                   rq/tensor_core.py:391-419
  plan_permutation / permute_fast  rq/tensor_core.py:81-151, 290-330
  permute_naive                    rq/tensor_core.py:271-273

Every numeric operation is a call into libqflex_b200.so (K1 permutation,
K2/K3 complex GEMM, K4 slicing).  PyTorch only owns the device buffers.

B200 design points
  * A contraction is `[batch] x (M x K) @ (K x N)` on the GEMM engine;
    operands are NOT permuted when the summed labels already form a
    contiguous prefix or suffix (the GEMM reads either layout, N or T), and
    the order of the summed index follows the larger operand so that the
    big intermediate is almost never touched by K1.
  * Labels that start with '@' are batch (hyper-)edges: kept, not summed,
    when shared.  The engine uses '@b' to batch many bit-strings through
    one plan walk as the GEMM batch dimension.
  * Buffers are flat 1-D torch tensors (rank-30 tensors exceed torch's
    dimension limit); `dims` carries the shape.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib

try:  # torch is plumbing only (device buffers + current stream)
    import torch
except ImportError:  # pragma: no cover
    torch = None

BATCH_PREFIX = "@"

_TORCH_OF = {}
_NP_OF = {}
if torch is not None:
    _TORCH_OF = {np.dtype(np.complex64): torch.complex64, np.dtype(np.complex128): torch.complex128}
    _NP_OF = {torch.complex64: np.dtype(np.complex64), torch.complex128: np.dtype(np.complex128)}

# fuse the big operand's permutation into the GEMM operand fetch (gathered A)
_gather_enabled = True


def set_gather(enabled: bool) -> bool:
    """Enable/disable gathered-A GEMMs in `contract`; returns the previous value."""
    global _gather_enabled
    prev, _gather_enabled = _gather_enabled, bool(enabled)
    return prev


# GEMM engine for contractions: "auto" (tcgen05 3xTF32 where it pays), "ffma", "tc3"
_GEMM_MODES = {"auto": _lib.GEMM_AUTO, "ffma": _lib.GEMM_FFMA, "tc3": _lib.GEMM_TC3}
_gemm_mode = _lib.GEMM_AUTO


def set_gemm_mode(mode: str) -> str:
    """Select the complex64 GEMM engine; returns the previous mode name."""
    global _gemm_mode
    if mode not in _GEMM_MODES:
        raise ValueError(f"gemm mode must be one of {sorted(_GEMM_MODES)}")
    prev = next(k for k, v in _GEMM_MODES.items() if v == _gemm_mode)
    _gemm_mode = _GEMM_MODES[mode]
    return prev


def tc3_real_macs_per_complex_mac(kernel: str = "cgemm_tc3k") -> int:
    """Real TF32 MMA multiply-adds a tensor-core kernel issues per complex
    multiply-add: the real-block form (`cgemm_tc3k`) 4 real products x 3
    (hi*hi + hi*lo + lo*hi) = 12, the Gauss form (`cgemm_tc3g`, and the
    128-column `cgemm_tc3w`) 3 x 3 = 9.  The 3xTF32 ceiling in algorithmic
    8-flop complex MACs is then TF32_peak * 8 / (2 * that)."""
    return 9 if kernel in ("cgemm_tc3g", "cgemm_tc3w") else 12


def get_gemm_mode() -> str:
    return next(k for k, v in _GEMM_MODES.items() if v == _gemm_mode)


def _require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("paper_1811_09599_b200 computes on a CUDA device; none is available "
                           "(there is no CPU fallback)")
    _lib.load()


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def device_buffer(n: int, dtype, device=None):
    _require_cuda()
    return torch.empty(max(int(n), 1), dtype=dtype, device=device or torch.cuda.current_device())


def _elem_bytes(t) -> int:
    return 8 if t.dtype == torch.complex64 else 16


class KernelTimer:
    """Collects CUDA-event timings of every library call made while active
    (bench.py's per-kernel roofline).  Each record: (kind, start, end,
    algorithmic flops, algorithmic bytes)."""

    def __init__(self):
        self.records = []

    def __enter__(self):
        global _timer
        self._prev = _timer
        _timer = self
        return self

    def __exit__(self, *exc):
        global _timer
        _timer = self._prev
        return False

    def summary(self, detail: bool = False, by_kernel: bool = False) -> dict:
        torch.cuda.synchronize()
        out: dict = {}
        for kind, a, b, flops, nbytes, *rest in self.records:
            if by_kernel:
                key = rest[1] if len(rest) > 1 and rest[1] else kind
            else:
                key = f"{kind} {rest[0]}" if detail and rest and rest[0] else kind
            d = out.setdefault(key, {"launches": 0, "ms": 0.0, "flops": 0, "bytes": 0})
            d["launches"] += 1
            d["ms"] += a.elapsed_time(b)
            d["flops"] += flops
            d["bytes"] += nbytes
        return out


_timer: Optional[KernelTimer] = None


class _timed:
    __slots__ = ("kind", "flops", "nbytes", "ev", "detail")

    def __init__(self, kind, flops=0, nbytes=0, detail=""):
        self.kind, self.flops, self.nbytes, self.detail = kind, flops, nbytes, detail

    def __enter__(self):
        if _timer is not None:
            self.ev = torch.cuda.Event(enable_timing=True)
            self.ev.record()
        return self

    def __exit__(self, *exc):
        if _timer is not None:
            end = torch.cuda.Event(enable_timing=True)
            end.record()
            kern = _lib.load().qf_last_kernel().decode()
            _timer.records.append((self.kind, self.ev, end, self.flops, self.nbytes, self.detail,
                                   kern))
        return False


# ---------------------------------------------------------------------------
# raw device ops on flat buffers


def permute_buffer(src, dims: Sequence[int], perm: Sequence[int], out=None):
    """out = ascontiguous(transpose(src.view(dims), perm)) on the device (K1)."""
    n = math.prod(dims)
    if out is None:
        out = device_buffer(n, src.dtype, src.device)
    with _timed("permute", 0, 2 * n * _elem_bytes(src),
                f"dims{tuple(dims)} perm{tuple(perm)}" if _timer else ""):
        st = _lib.load().qf_permute(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                    len(dims), _lib.dims_array(dims), _lib.perm_array(perm),
                                    _elem_bytes(src), stream_handle())
    _lib.check(st, "permute")
    return out


def fix_buffer(src, dims: Sequence[int], axis: int, value: int):
    """src[..., value, ...] along `axis`, contiguous (K4)."""
    outer = math.prod(dims[:axis])
    inner = math.prod(dims[axis + 1:])
    out = device_buffer(outer * inner, src.dtype, src.device)
    st = _lib.load().qf_fix_axis(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                 outer, int(dims[axis]), inner, int(value), _elem_bytes(src),
                                 stream_handle())
    _lib.check(st, "fix")
    return out


def gather_buffer(src, dims: Sequence[int], axis: int, idx):
    """dst[b, ...] = src[..., idx[b], ...] (K4, batched); idx: device int32."""
    outer = math.prod(dims[:axis])
    inner = math.prod(dims[axis + 1:])
    nidx = int(idx.numel())
    out = device_buffer(outer * inner * nidx, src.dtype, src.device)
    st = _lib.load().qf_gather_axis(ctypes.c_void_p(src.data_ptr()),
                                    ctypes.c_void_p(out.data_ptr()), outer, int(dims[axis]), inner,
                                    ctypes.c_void_p(idx.data_ptr()), nidx, _elem_bytes(src),
                                    stream_handle())
    _lib.check(st, "gather")
    return out


def affine_offsets(out, n: int, rep: int, entry: int, base=None, stride: int = 0):
    """out[e] = (base[e // rep] if base is given else (e // rep) * entry)
    + (e % rep) * stride on the device (int64 entry-base tables)."""
    st = _lib.load().qf_affine_offsets(ctypes.c_void_p(out.data_ptr()), int(n), int(rep),
                                       int(entry),
                                       ctypes.c_void_p(base.data_ptr()) if base is not None else None,
                                       int(stride), stream_handle())
    _lib.check(st, "affine_offsets")


def zero_buffer(y):
    """y[:] = 0 (stream-ordered memset)."""
    st = _lib.load().qf_fill_zero(ctypes.c_void_p(y.data_ptr()), int(y.numel()) * _elem_bytes(y),
                                  stream_handle())
    _lib.check(st, "fill_zero")


def accumulate_buffer(x, y, n: Optional[int] = None):
    """y[:n] += x[:n] (K5)."""
    n = int(x.numel()) if n is None else int(n)
    st = _lib.load().qf_accumulate(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), n,
                                   _elem_bytes(y), stream_handle())
    _lib.check(st, "accumulate")


def gemm_buffer(batch, M, N, K, A, opA, B, opB, C, alpha=1.0, beta=0.0, mode=None):
    """C[b] = alpha op(A[b]) op(B[b]) + beta C[b] on flat row-major buffers."""
    lda = K if opA == _lib.OP_N else M
    ldb = N if opB == _lib.OP_N else K
    lib = _lib.load()
    sA, sB, sC = M * K, K * N, M * N
    eb = _elem_bytes(C)
    with _timed("gemm", 8 * batch * M * N * K, eb * batch * (sA + sB + sC),
                f"b{batch} m{M} n{N} k{K} {'NT'[opA]}{'NT'[opB]}" if _timer else ""):
        st = _gemm_call(lib, batch, M, N, K, A, lda, opA, B, ldb, opB, C, sA, sB, sC, alpha, beta,
                        mode)
    _lib.check(st, "gemm")


_GATHER_TABLES: dict = {}


def _gather_tables(dims, labels, rows, cols, device):
    """Device int32 offset tables of a tensor's free (`rows`) and summed
    (`cols`) label groups inside one batch entry (memoised per layout)."""
    key = (tuple(dims), tuple(labels), tuple(rows), tuple(cols), str(device))
    hit = _GATHER_TABLES.get(key)
    if hit is not None:
        return hit
    stride = {}
    acc = 1
    for l, d in zip(reversed(labels), reversed(dims)):
        stride[l] = acc
        acc *= d
    dim = dict(zip(labels, dims))

    def table(group):
        off = np.zeros(1, dtype=np.int64)
        for l in group:
            off = (off[:, None] + np.arange(dim[l], dtype=np.int64)[None, :] * stride[l]).reshape(-1)
        return off

    r, c = table(rows), table(cols)
    # consecutive rows adjacent in memory: the K3 engines then fetch lane = row
    rows_unit = bool(r.size > 1 and r[1] - r[0] == 1)
    hit = (torch.from_numpy(r.astype(np.int32)).to(device),
           torch.from_numpy(c.astype(np.int32)).to(device), rows_unit)
    if len(_GATHER_TABLES) > 512:
        _GATHER_TABLES.clear()
    _GATHER_TABLES[key] = hit
    return hit


def gemm_gather_buffer(batch, M, N, K, A, sA, roff, coff, B, opB, C, mode=None, rows_unit=False):
    """C[b] = A_gathered[b] @ op(B[b]) (complex64): the big operand is read
    through offset tables instead of being transposed first.  `rows_unit`
    (roff[r] = roff[0] + r) is a fetch-direction hint for the engines."""
    ldb = N if opB == _lib.OP_N else K
    lib = _lib.load()
    flags = _lib.GATHER_ROWS_UNIT if rows_unit else 0
    with _timed("gemm", 8 * batch * M * N * K, 8 * batch * (M * K + K * N + M * N),
                f"b{batch} m{M} n{N} k{K} G{'NT'[opB]}" if _timer else ""):
        st = lib.qf_cgemm_c64_gather((_gemm_mode if mode is None else mode) | flags, batch, M, N, K,
                                     ctypes.c_void_p(A.data_ptr()), sA,
                                     ctypes.c_void_p(roff.data_ptr()),
                                     ctypes.c_void_p(coff.data_ptr()),
                                     ctypes.c_void_p(B.data_ptr()), max(ldb, 1), K * N, opB,
                                     ctypes.c_void_p(C.data_ptr()), max(N, 1), M * N,
                                     1.0, 0.0, 0.0, 0.0, stream_handle())
    _lib.check(st, "gemm_gather")


def _gemm_call(lib, batch, M, N, K, A, lda, opA, B, ldb, opB, C, sA, sB, sC, alpha, beta, mode):
    if C.dtype == torch.complex64:
        st = lib.qf_cgemm_c64(_gemm_mode if mode is None else mode, batch, M, N, K,
                              ctypes.c_void_p(A.data_ptr()), max(lda, 1), sA, opA,
                              ctypes.c_void_p(B.data_ptr()), max(ldb, 1), sB, opB,
                              ctypes.c_void_p(C.data_ptr()), max(N, 1), sC,
                              float(np.real(alpha)), float(np.imag(alpha)),
                              float(np.real(beta)), float(np.imag(beta)), stream_handle())
    else:
        st = lib.qf_zgemm_c128(batch, M, N, K,
                               ctypes.c_void_p(A.data_ptr()), max(lda, 1), sA, opA,
                               ctypes.c_void_p(B.data_ptr()), max(ldb, 1), sB, opB,
                               ctypes.c_void_p(C.data_ptr()), max(N, 1), sC,
                               float(np.real(alpha)), float(np.imag(alpha)),
                               float(np.real(beta)), float(np.imag(beta)), stream_handle())
    return st


# ---------------------------------------------------------------------------
# labelled device tensor


class Tensor:
    """A row-major device tensor with one string label per index.

    `array` (numpy) may be passed instead of a device buffer; it is
    uploaded once.  `.array` downloads a numpy copy (API compatibility with
    the reference's numpy-backed Tensor)."""

    __slots__ = ("labels", "_data", "dims", "_layouts", "_view")

    def __init__(self, labels: Sequence[str], array, dims: Optional[Sequence[int]] = None):
        labels = tuple(labels)
        if len(set(labels)) != len(labels):
            raise ValueError(f"duplicate labels: {labels}")
        if isinstance(array, np.ndarray) or np.isscalar(array):
            arr = np.asarray(array)
            if arr.dtype not in _TORCH_OF:
                # real/integer input widens without rounding: 8-byte reals to
                # complex128, everything narrower to complex64 (the reference
                # keeps any numpy dtype; values compare equal either way)
                wide = arr.dtype.kind in "fiu" and arr.dtype.itemsize >= 8
                arr = arr.astype(np.complex128 if wide else np.complex64)
            dims = arr.shape
            _require_cuda()
            data = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).to(
                torch.cuda.current_device())
        else:
            data = array
            if dims is None:
                dims = tuple(array.shape)
            data = data.reshape(-1)
        dims = tuple(int(d) for d in dims)
        if len(dims) != len(labels):
            raise ValueError(f"{len(dims)}-d array with {len(labels)} labels")
        self.labels = labels
        self._data = data
        self.dims = dims
        self._layouts = None  # memoised transposes (labels -> Tensor)
        self._view = None     # (base, label, value) of a lazy fix (see fix_view)

    @property
    def data(self):
        """Flat device buffer (a lazy fix view is materialised on first use)."""
        d = self._data
        if d is None:
            base, label, value = self._view
            d = fix_buffer(base.data, base.dims, base.labels.index(label), value)
            self._data = d
        return d

    @data.setter
    def data(self, value):
        self._data = value

    @property
    def buf(self):
        """The storage (for dtype/device queries); never materialises a view."""
        return self._data if self._data is not None else self._view[0].buf

    def raw(self):
        """(buffer, element offset, stride of the leading index) -- a view's
        entries along its leading (batch) index are contiguous blocks of the
        base buffer; a plain tensor is (data, 0, entry size)."""
        if self._data is not None or self._view is None:
            lead = self.dims[0] if self.dims else 1
            return self.data, 0, self.size // max(lead, 1)
        base, label, value = self._view
        ax = base.labels.index(label)
        block = math.prod(base.dims[ax + 1:])
        return base.data, value * block, base.dims[ax] * block if ax == 1 else 0

    def fix_view(self, label: str, value: int) -> "Tensor":
        """`fix` without a copy when the fixed index is the outermost one or
        directly follows a leading batch axis: the result is a strided view
        (each batch entry a contiguous block) that the late-slicing GEMMs read
        in place; any other use materialises it.  Otherwise a plain fix."""
        ax = self.labels.index(label)
        if self._view is not None or not (ax == 0 or (ax == 1 and _is_batch(self.labels[0]))):
            return self.fix(label, value)
        if not 0 <= value < self.dims[ax]:
            raise ValueError(f"value {value} out of range for {label!r} (dim {self.dims[ax]})")
        t = Tensor.__new__(Tensor)
        t.labels = self.labels[:ax] + self.labels[ax + 1:]
        t.dims = self.dims[:ax] + self.dims[ax + 1:]
        t._data = None
        t._layouts = None
        t._view = (self, label, int(value))
        return t

    @property
    def size(self) -> int:
        return math.prod(self.dims)

    @property
    def nbytes(self) -> int:
        return self.size * _elem_bytes(self.buf)

    @property
    def dtype(self):
        return _NP_OF[self.buf.dtype]

    @property
    def array(self) -> np.ndarray:
        flat = self.data[: self.size].cpu().numpy()
        return flat.reshape(self.dims) if self.dims else flat.reshape(())

    def dim_of(self, label: str) -> int:
        return self.dims[self.labels.index(label)]

    def relabel(self, mapping: dict) -> "Tensor":
        return Tensor(tuple(mapping.get(l, l) for l in self.labels), self.data, self.dims)

    def fix(self, label: str, value: int) -> "Tensor":
        """Slice one index to a fixed value, dropping it (device gather)."""
        ax = self.labels.index(label)
        if not 0 <= value < self.dims[ax]:
            raise ValueError(f"value {value} out of range for {label!r} (dim {self.dims[ax]})")
        out = fix_buffer(self.data, self.dims, ax, value)
        return Tensor(self.labels[:ax] + self.labels[ax + 1:], out,
                      self.dims[:ax] + self.dims[ax + 1:])

    def gather(self, label: str, idx, batch_label: str = "@b") -> "Tensor":
        """Batch slice: new leading `batch_label` axis, entry b = fix(label, idx[b])."""
        ax = self.labels.index(label)
        out = gather_buffer(self.data, self.dims, ax, idx)
        return Tensor((batch_label,) + self.labels[:ax] + self.labels[ax + 1:], out,
                      (int(idx.numel()),) + self.dims[:ax] + self.dims[ax + 1:])

    def transpose_to(self, labels: Sequence[str], thread_count: int = 1) -> "Tensor":
        labels = tuple(labels)
        if labels == self.labels:
            return self
        if self._layouts is not None and labels in self._layouts:
            return self._layouts[labels]
        if sorted(labels) != sorted(self.labels):
            raise ValueError(f"{labels} is not a permutation of {self.labels}")
        perm = [self.labels.index(l) for l in labels]
        out = permute_buffer(self.data, self.dims, perm)
        t = Tensor(labels, out, tuple(self.dims[p] for p in perm))
        # an intermediate reused across paths (reuse=global/outer steps) is
        # permuted once, not once per path; the copy dies with its source
        if self._layouts is None:
            self._layouts = {}
        self._layouts[labels] = t
        return t

    def scalar(self) -> complex:
        if self.labels:
            raise ValueError(f"tensor still has indexes {self.labels}")
        return complex(self.data[0].item())

    def __repr__(self):
        return f"Tensor({self.labels}, dims={self.dims}, dtype={self.dtype}, device)"


def _is_batch(label: str) -> bool:
    return label.startswith(BATCH_PREFIX)


@dataclass(frozen=True)
class ContractShape:
    """GEMM view of one pairwise contraction (per batch entry)."""

    batch: int
    m: int
    k: int
    n: int

    @property
    def flops(self) -> int:
        """Reference convention: 8 real ops per complex multiply-add,
        counted per batch entry (rq/contraction_plan.py:516)."""
        return 8 * self.m * self.k * self.n


def contract_shape(a: Tensor, b: Tensor, skip=()) -> ContractShape:
    """Per-entry GEMM view.  Labels in `skip` (open outputs whose slicing is
    deferred, see LateBits) count like batch labels: not part of m or n."""
    bset, aset = set(b.labels), set(a.labels)
    bt = m = k = 1
    for l, d in zip(a.labels, a.dims):
        if _is_batch(l) or l in skip:   # batch axes count per entry, shared or not
            bt *= d
        elif l in bset:
            k *= d
        else:
            m *= d
    n = 1
    for l, d in zip(b.labels, b.dims):
        if l in aset:
            continue
        if _is_batch(l) or l in skip:
            bt *= d
        else:
            n *= d
    return ContractShape(bt, m, k, n)


# measured B200 rates (scripts/gemm_bench.py, bench.py --workload permute):
# gathered-A tensor-core GEMMs ~140 TFLOP/s at long K, plain strided ones fed
# by TMA ~205 TFLOP/s, the permutation ~5.5 TB/s, GEMM operand streams ~5 TB/s
_RATE_GATHER, _RATE_TMA, _RATE_PERMUTE, _RATE_HBM = 140e12, 205e12, 5.5e12, 5.0e12


def _permute_pays(bt: int, m: int, k: int, n: int) -> bool:
    """For compute-bound shapes a separate permute of the big operand plus
    the TMA-fed GEMM beats fetching it through offset tables."""
    if k < 128 or n < 128:
        return False
    flops = 8.0 * bt * m * k * n
    nbytes = 8.0 * bt * (m * k + k * n + m * n)
    t_gather = max(flops / _RATE_GATHER, nbytes / _RATE_HBM)
    t_perm = 16.0 * bt * m * k / _RATE_PERMUTE + max(flops / _RATE_TMA, nbytes / _RATE_HBM)
    return t_perm < t_gather


def _a_view(labels, dims, a_free, k_order):
    """The big operand's per-entry layout as a TMA-describable view, or None:
    its summed labels in at most two runs of adjacent labels, the inner run
    innermost and contiguous (kin entries, kin % 8 == 0), and its free labels
    (in memory order) in at most two runs around the outer summed run.
    -> (kin, rows_a, s_rows_a, kout, s_kout, rows_b, s_rows_b) in elements
    (see qf_cgemm_c64_view)."""
    if not k_order or not labels or labels[-1] != k_order[-1]:
        return None
    if [l for l in labels if l not in k_order] != list(a_free):
        return None
    if [l for l in labels if l in k_order] != list(k_order):
        return None
    dim = dict(zip(labels, dims))
    stride, acc = {}, 1
    for l, d in zip(reversed(labels), reversed(dims)):
        stride[l] = acc
        acc *= d
    ks = set(k_order)
    runs, prev = [], None                 # runs of adjacent summed labels
    for p, l in enumerate(labels):
        if l in ks:
            if prev is not None and prev == p - 1:
                runs[-1].append(l)
            else:
                runs.append([l])
            prev = p
    if len(runs) > 2:
        return None
    inner = runs[-1]
    kin = math.prod(dim[l] for l in inner)
    if kin % 8:
        return None
    first_inner = labels.index(inner[0])
    if len(runs) == 2:
        outer = runs[0]
        p0, p1 = labels.index(outer[0]), labels.index(outer[-1])
        run_b, run_a = labels[:p0], labels[p1 + 1:first_inner]
        kout, s_kout = math.prod(dim[l] for l in outer), stride[outer[-1]]
    else:
        run_b, run_a = (), labels[:first_inner]
        kout, s_kout = 1, kin
    if not run_a:
        return None            # summed labels contiguous: a plain layout
    rows_a = math.prod(dim[l] for l in run_a)
    s_rows_a = stride[run_a[-1]]
    rows_b = math.prod(dim[l] for l in run_b) if run_b else 1
    s_rows_b = stride[run_b[-1]] if run_b else acc
    if not (rows_a % 128 == 0 if rows_a >= 128 else 128 % rows_a == 0):
        return None
    if any(x % 2 for x in (s_rows_a, s_kout, s_rows_b)):
        return None
    return kin, rows_a, s_rows_a, kout, s_kout, rows_b, s_rows_b


def _a_tview(labels, dims, a_free, k_order):
    """The big operand's per-entry layout as a TRANSPOSED TMA view, or None:
    its innermost label free, the free labels in at most two runs (the inner
    one contiguous) and the summed labels in at most two runs, in any
    interleaving -> (rows_a, rows_b, s_rows_b, kin, s_kin, kout, s_kout) in
    elements (see qf_cgemm_c64_tview)."""
    if not labels or not k_order or labels[-1] in k_order:
        return None
    ks = set(k_order)
    if [l for l in labels if l not in ks] != list(a_free) or [l for l in labels if l in ks] != list(k_order):
        return None
    stride, acc = {}, 1
    for l, d in zip(reversed(labels), reversed(dims)):
        stride[l] = acc
        acc *= d
    dim = dict(zip(labels, dims))
    runs = []                      # (summed?, [labels]) outermost first
    for l in labels:
        t = l in ks
        if runs and runs[-1][0] == t:
            runs[-1][1].append(l)
        else:
            runs.append((t, [l]))
    free = [r for t, r in runs if not t]
    summ = [r for t, r in runs if t]
    if len(free) > 2 or len(summ) > 2:
        return None
    size = lambda r: math.prod(dim[l] for l in r)
    rows_a = size(free[-1])
    rows_b, s_rows_b = (size(free[0]), stride[free[0][-1]]) if len(free) == 2 else (1, acc)
    kin, s_kin = size(summ[-1]), stride[summ[-1][-1]]
    kout, s_kout = (size(summ[0]), stride[summ[0][-1]]) if len(summ) == 2 else (1, acc)
    if kin % 8 or rows_a % 2 or not (rows_a % 128 == 0 if rows_a >= 128 else 128 % rows_a == 0):
        return None
    if any(x % 2 for x in (s_rows_b, s_kin, s_kout)):
        return None
    return rows_a, rows_b, s_rows_b, kin, s_kin, kout, s_kout


def _gemm_view(nb, m, n, k, a_ptr, strideA, view, B, ldb, sB, opB, out, b_boff=None,
               b_nslice=0) -> bool:
    """Run the TMA-fed kernel on a view of the big operand; False if the
    library reports the shape/view unsupported (caller falls back)."""
    if _gemm_mode == _lib.GEMM_FFMA or strideA % 2 or not _view_enabled:
        return False
    kin, ra, sra, ko, sko, rb, srb = view
    lib = _lib.load()
    with _timed("gemm", 8 * nb * m * n * k, 8 * nb * (m * k + k * n + m * n),
                f"b{nb} m{m} n{n} k{k} V{'NT'[opB]}" if _timer else ""):
        st = lib.qf_cgemm_c64_view(
            _gemm_mode, nb, m, n, k, ctypes.c_void_p(a_ptr), strideA, kin, ra, sra, ko, sko, rb,
            srb, ctypes.c_void_p(B.data.data_ptr()), ldb, sB, opB,
            ctypes.c_void_p(b_boff.data_ptr() if b_boff is not None else 0), int(b_nslice),
            ctypes.c_void_p(out.data_ptr()), max(n, 1), m * n, 1.0, 0.0, 0.0, 0.0, stream_handle())
    if st == _lib.QF_ERR_UNSUPPORTED:
        return False
    _lib.check(st, "gemm_view")
    return True


def _gemm_tview(nb, m, n, k, a: "Tensor", strideA, a_free, k_order, B, ldb, sB, opB, out) -> bool:
    """Run the TMA-fed kernel on a TRANSPOSED view of the big operand (its
    innermost labels free; long K: the wide kernel); False if the layout has
    no such view or the library reports it unsupported (caller falls back)."""
    if _gemm_mode == _lib.GEMM_FFMA or strideA % 2 or not (_view_enabled and _tview_enabled):
        return False
    off = len(a.labels) - len(a_free) - len(k_order)        # leading batch labels
    tv = _a_tview(a.labels[off:], a.dims[off:], a_free, k_order)
    if tv is None:
        return False
    ra, rb, srb, kin, ski, ko, sko = tv
    with _timed("gemm", 8 * nb * m * n * k, 8 * nb * (m * k + k * n + m * n),
                f"b{nb} m{m} n{n} k{k} TV{'NT'[opB]}" if _timer else ""):
        st = _lib.load().qf_cgemm_c64_tview(
            _gemm_mode, nb, m, n, k, ctypes.c_void_p(a.data.data_ptr()), strideA, ra, rb, srb, kin,
            ski, ko, sko, ctypes.c_void_p(B.data.data_ptr()), ldb, sB, opB, ctypes.c_void_p(0), 0,
            ctypes.c_void_p(out.data_ptr()), max(n, 1), m * n, 1.0, 0.0, 0.0, 0.0, stream_handle())
    if st == _lib.QF_ERR_UNSUPPORTED:
        return False
    _lib.check(st, "gemm_tview")
    return True


_view_enabled = True
_tview_enabled = True
_compute_views = True   # A/B knob: TMA views for compute-bound shapes too (contract)


def set_tview(enabled: bool) -> bool:
    """Enable/disable transposed (rows-innermost) TMA views; returns the previous value."""
    global _tview_enabled
    prev, _tview_enabled = _tview_enabled, bool(enabled)
    return prev


def set_view(enabled: bool) -> bool:
    """Enable/disable TMA-fed strided views of the big operand; returns the previous value."""
    global _view_enabled
    prev, _view_enabled = _view_enabled, bool(enabled)
    return prev


def contract(a: Tensor, b: Tensor, thread_count: int = 1, mu: int = 5, nu: int = 10,
             front=(), tail=()) -> Tensor:
    """Contract over all shared labels (batch '@' labels are kept).

    Output labels: batch labels (a's order), then a's free labels, then
    b's free labels -- the reference's a_free + b_free order
    (rq/tensor_core.py:396-419) with the batch axis in front.  Labels in
    `front` (open outputs awaiting a late slice) are moved to the front of
    their operand's free group when that costs no extra pass (gathered big
    operand; memoised small-operand layout), so a later per-bit-string slice
    reads long contiguous runs.  Labels in `tail` (those of the operand this
    result meets next) go last among the small operand's free labels, so the
    next contraction finds a summed label innermost (TMA-fed view)."""
    if a.buf.dtype != b.buf.dtype:
        raise ValueError(f"dtype mismatch: {a.dtype} vs {b.dtype}")
    if b.size > a.size:
        # the big operand goes first (its layout decides the GEMM); the output
        # is then [batch, b_free, a_free] -- labels carry the order
        a, b = b, a
    bset, aset = set(b.labels), set(a.labels)
    batch = [l for l in a.labels if l in bset and _is_batch(l)]
    shared_a = [l for l in a.labels if l in bset and not _is_batch(l)]
    for l in batch + shared_a:
        if a.dim_of(l) != b.dim_of(l):
            raise ValueError(f"dimension mismatch on {l!r}: {a.dim_of(l)} vs {b.dim_of(l)}")
    a_free = [l for l in a.labels if l not in bset]
    b_free = [l for l in b.labels if l not in aset]
    if front:
        b_free = [l for l in b_free if l in front] + [l for l in b_free if l not in front]
    if tail:
        b_free = [l for l in b_free if l not in tail] + [l for l in b_free if l in tail]
    # summed-index order follows the bigger operand so it is not permuted
    if a.size >= b.size:
        k_order = shared_a
    else:
        k_order = [l for l in b.labels if l in aset and not _is_batch(l)]

    def operand(t: Tensor, free, first_is_free):
        n_layout = batch + (free + k_order if first_is_free else k_order + free)
        t_layout = batch + (k_order + free if first_is_free else free + k_order)
        if list(t.labels) == n_layout:
            return t, _lib.OP_N
        if list(t.labels) == t_layout:
            return t, _lib.OP_T
        return t.transpose_to(n_layout), _lib.OP_N

    bt = math.prod(a.dim_of(l) for l in batch)
    m = math.prod(a.dim_of(l) for l in a_free)
    k = math.prod(a.dim_of(l) for l in k_order)
    n = math.prod(b.dim_of(l) for l in b_free)
    out = device_buffer(bt * m * n, a.data.dtype, a.data.device)
    B, opB = operand(b, b_free, False)     # N: [batch][K][N], T: [batch][N][K]
    a_n = batch + a_free + k_order
    a_t = batch + k_order + a_free
    entry = a.size // max(bt, 1)
    nb = len(batch)
    ldb = n if opB == _lib.OP_N else k
    scattered = (list(a.labels) not in (a_n, a_t) and a.data.dtype == torch.complex64
                 and list(a.labels[:nb]) == batch and entry >= 4096 and _gather_enabled)
    # A strided view read by TMA costs nothing over a plain layout: taken
    # whenever the layout has one, compute-bound shapes included (config 5:
    # the 16^7-entry operands of the region builds were permuted first,
    # 0.7 ms each, 18% of a path).
    view = _a_view(a.labels[nb:], a.dims[nb:], a_free, k_order) if scattered else None
    if view is not None and not _compute_views and _permute_pays(bt, m, k, n):
        view = None
    if view is not None and _gemm_view(bt, m, n, k, a.data.data_ptr(), entry, view, B,
                                       max(ldb, 1), k * n, opB, out):
        pass
    elif (view is None and scattered and _compute_views and k >= 256 and n >= 128
            and _gemm_tview(bt, m, n, k, a, entry, a_free, k_order, B, max(ldb, 1), k * n, opB,
                            out)):
        pass     # rows innermost: a transposed TMA view on the wide long-K kernel
    elif (scattered and entry < 2 ** 31 and m <= 2 ** 22 and k <= 4096
            and not _permute_pays(bt, m, k, n)):
        # no view: fuse the big operand's permutation into the GEMM fetch
        # through offset tables (memory-bound shapes only)
        if front:
            a_free = [l for l in a_free if l in front] + [l for l in a_free if l not in front]
        roff, coff, rows_unit = _gather_tables(a.dims[nb:], a.labels[nb:], a_free, k_order,
                                               a.data.device)
        gemm_gather_buffer(bt, m, n, k, a.data, entry, roff, coff, B.data, opB, out,
                           rows_unit=rows_unit)
    else:
        if front and list(a.labels) not in (a_n, a_t):   # permuted anyway
            a_free = [l for l in a_free if l in front] + [l for l in a_free if l not in front]
        A, opA = operand(a, a_free, True)  # N: [batch][M][K], T: [batch][K][M]
        gemm_buffer(bt, m, n, k, A.data, opA, B.data, opB, out)
    labels = tuple(batch + a_free + b_free)
    dims = tuple(a.dim_of(l) for l in batch + a_free) + tuple(b.dim_of(l) for l in b_free)
    return Tensor(labels, out, dims)


# ---------------------------------------------------------------------------
# late output batching


def _strides(t: Tensor) -> dict:
    out, acc = {}, 1
    for l, d in zip(reversed(t.labels), reversed(t.dims)):
        out[l] = acc
        acc *= d
    return out


_ROW_TABLES: dict = {}


def _outer_table(dims, labels, outer, device):
    """int64 offsets of the `outer` label group (row-major over `outer`)."""
    key = (tuple(dims), tuple(labels), tuple(outer), str(device))
    hit = _ROW_TABLES.get(key)
    if hit is None:
        stride = {}
        acc = 1
        for l, d in zip(reversed(labels), reversed(dims)):
            stride[l] = acc
            acc *= d
        dim = dict(zip(labels, dims))
        off = np.zeros(1, dtype=np.int64)
        for l in outer:
            off = (off[:, None] + np.arange(dim[l], dtype=np.int64)[None, :] * stride[l]).reshape(-1)
        hit = torch.from_numpy(off).to(device)
        if len(_ROW_TABLES) > 256:
            _ROW_TABLES.clear()
        _ROW_TABLES[key] = hit
    return hit


class LateBits:
    """Bit-strings whose output slicing is deferred ("late output batching").

    The reference fixes every output index before contracting
    (Net2D.fix_outputs, rq/network_builder.py:134-149).  For a batch of B
    bit-strings the early plan steps touch only a few qubits, so this keeps
    those `out` indices OPEN -- computing all 2^q combinations once instead
    of B copies -- and slices the batch out (Tensor.fix per bit-string,
    rq/tensor_core.py:366-372) only when 2^q would exceed `limit` (default
    B/2).  Same products and sums per amplitude, in a different grouping.

    bits_t: DEVICE int32 (rows, B) matrix; `rows` maps an out label to its
    row.  The slice is either fused into the next GEMM's operand fetch
    (qf_cgemm_c64_gather_boff) or materialised (qf_gather_rows)."""

    def __init__(self, bits_t, rows: dict, limit: Optional[int] = None, label: str = "@b"):
        if bits_t.dtype != torch.int32 or bits_t.dim() != 2 or not bits_t.is_contiguous():
            raise ValueError("bits must be a contiguous 2-D int32 device tensor")
        self.bits_t = bits_t
        self.rows = dict(rows)
        self.nb = int(bits_t.shape[1])
        self.limit = max(1, self.nb // 2) if limit is None else int(limit)
        self.label = label

    def outs(self, t: Tensor) -> list:
        return [l for l in t.labels if l in self.rows]

    def offsets(self, t: Tensor, outs) -> "torch.Tensor":
        """Per-entry element offsets of the bit-strings' slice of `t`."""
        st = _strides(t)
        off = torch.empty(max(self.nb, 1), dtype=torch.int64, device=t.buf.device)
        rows = (_i32 * max(1, len(outs)))(*[self.rows[l] for l in outs])
        strides = (ctypes.c_int64 * max(1, len(outs)))(*[st[l] for l in outs])
        with _timed("gather", 0, 4 * self.nb * (len(outs) + 2), "bit_offsets" if _timer else ""):
            rc = _lib.load().qf_bit_offsets(ctypes.c_void_p(self.bits_t.data_ptr()), self.nb,
                                            len(outs), rows, strides, self.nb,
                                            ctypes.c_void_p(off.data_ptr()), stream_handle())
        _lib.check(rc, "bit_offsets")
        return off

    def batch(self, t: Tensor) -> Tensor:
        """Slice the batch out of `t`'s open outputs: new leading batch axis."""
        outs = self.outs(t)
        if not outs:
            return t
        if self.label in t.labels:
            raise ValueError(f"tensor already has batch label {self.label!r}")
        oset = set(outs)
        rest = [(l, d) for l, d in zip(t.labels, t.dims) if l not in oset]
        inner = 0
        while inner < len(t.labels) and t.labels[len(t.labels) - 1 - inner] not in oset:
            inner += 1
        L = math.prod(t.dims[len(t.dims) - inner:]) if inner else 1
        outer = [l for l in t.labels[:len(t.labels) - inner] if l not in oset]
        per = math.prod(d for _, d in rest)
        off = self.offsets(t, outs)
        n_outer = per // L
        ooff = (_outer_table(t.dims, t.labels, outer, t.data.device) if outer else None)
        out = device_buffer(self.nb * per, t.data.dtype, t.data.device)
        eb = _elem_bytes(t.data)
        with _timed("gather", 0, 2 * eb * self.nb * per,
                    f"late rows b{self.nb} x{n_outer} L{L}" if _timer else ""):
            rc = _lib.load().qf_gather_rows(ctypes.c_void_p(t.data.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), self.nb,
                                            ctypes.c_void_p(off.data_ptr()), n_outer,
                                            ctypes.c_void_p(ooff.data_ptr() if ooff is not None
                                                            else 0), L, eb, stream_handle())
        _lib.check(rc, "gather_rows")
        return Tensor((self.label,) + tuple(l for l, _ in rest), out,
                      (self.nb,) + tuple(d for _, d in rest))

    def _batched_size(self, t: Tensor) -> int:
        outs = self.outs(t)
        return t.size // (1 << len(outs)) * self.nb if outs else t.size


_i32 = ctypes.c_int32


def contract_late(a: Tensor, b: Tensor, late: LateBits, tail=(), lead=()) -> Tensor:
    """`contract` for networks whose outputs are sliced late (LateBits).

    Both operands without a batch axis and few open outputs between them:
    an ordinary contraction (the outputs are free indices).  Otherwise the
    open outputs are sliced to the batch first -- for the bigger operand
    fused into the GEMM's gathered operand fetch when it can be."""
    oa, ob = late.outs(a), late.outs(b)
    if not oa and not ob:
        return contract(a, b, tail=tail)
    lb = late.label
    if lb not in a.labels and lb not in b.labels and 2 ** (len(oa) + len(ob)) <= late.limit:
        r = _contract_open(a, b, late, tail)
        return r if r is not None else contract(a, b, front=late.rows, tail=tail)
    big, small = (a, b) if late._batched_size(a) >= late._batched_size(b) else (b, a)
    fused = _contract_sliced(big, small, late, tail, lead)
    if fused is not None:
        return fused
    big, small = late.batch(big), late.batch(small)
    return contract(big, small, tail=tail)


_ZEROS: dict = {}


def _zero_offsets(n: int, device):
    key = (n, str(device))
    z = _ZEROS.get(key)
    if z is None:
        z = _ZEROS[key] = torch.empty(max(n, 1), dtype=torch.int64, device=device)
        affine_offsets(z, n, 1, 0)
    return z


def _row_blocks(big: Tensor, a_free, k_order, n: int) -> Optional[int]:
    """Rows per block when `big` is laid out [outer free][summed][inner free]
    with the free labels in memory order (so A(r, k) = (r / rin) * rin*K +
    r % rin + k*rin, qf_cgemm_c64_rowblocks), the summed labels contiguous
    and in the GEMM's k order, and the shape within the row engines' range."""
    if big.buf.dtype != torch.complex64 or not k_order or n > 16:
        return None
    labels = list(big.labels)
    ks = labels.index(k_order[0])
    if labels[ks:ks + len(k_order)] != list(k_order):
        return None
    if labels[:ks] + labels[ks + len(k_order):] != list(a_free):
        return None
    inner = labels[ks + len(k_order):]
    if not inner:
        return None
    rin = math.prod(big.dim_of(l) for l in inner)
    k = math.prod(big.dim_of(l) for l in k_order)
    if rin % 32 or k * n > 4096:
        return None
    return rin


def _contract_open(a: Tensor, b: Tensor, late: LateBits, tail=()) -> Optional[Tensor]:
    """Both operands with open outputs, no batch axis yet: the smaller
    operand's open outputs become the GEMM batch (its slices side by side,
    the big operand broadcast through all-zero entry offsets and read
    through gathered tables), so the result keeps EVERY open output in
    front: [small's outs, big's outs, rows, cols].  A later per-bit-string
    slice is then one contiguous block per entry.  None if not eligible."""
    big, small = (a, b) if a.size >= b.size else (b, a)
    so = late.outs(small)
    if (not so or big.buf.dtype != torch.complex64 or not _gather_enabled
            or big.size >= 2 ** 31):
        return None
    sset, bset = set(small.labels), set(big.labels)
    if any(_is_batch(l) for l in sset | bset):
        return None
    k_order = [l for l in big.labels if l in sset]
    front = set(late.rows)
    a_free = [l for l in big.labels if l not in sset]
    a_free = [l for l in a_free if l in front] + [l for l in a_free if l not in front]
    s_free = [l for l in small.labels if l not in bset and l not in so]
    s_free = [l for l in s_free if l not in tail] + [l for l in s_free if l in tail]
    for l in k_order:
        if big.dim_of(l) != small.dim_of(l):
            raise ValueError(f"dimension mismatch on {l!r}: {big.dim_of(l)} vs {small.dim_of(l)}")
    m = math.prod(big.dim_of(l) for l in a_free)
    k = math.prod(big.dim_of(l) for l in k_order)
    n = math.prod(small.dim_of(l) for l in s_free)
    if k > 4096 or k == 0:
        return None
    nbat = 1 << len(so)
    B = small.transpose_to(tuple(so + k_order + s_free))    # [outs][K][N]
    out = device_buffer(nbat * m * n, big.data.dtype, big.data.device)
    lib = _lib.load()
    detail = f"b{nbat} m{m} n{n} k{k} O" if _timer else ""
    if _timer is not None and os.environ.get("QF_DEBUG_LAYOUT"):
        detail += f" BIG{list(zip(big.labels, big.dims))} free{a_free} k{k_order} SMALL{list(zip(small.labels, small.dims))} so{so} sfree{s_free}"
    st = None
    view = (_a_view(big.labels, big.dims, a_free, k_order)
            if 32 <= k <= 128 and n > 32 and m >= 65536 and _view_enabled
            and _gemm_mode != _lib.GEMM_FFMA
            else None)
    if view is not None:
        # big operand as a TMA-fed strided view (summed labels split around a
        # free run), one launch per open output of the small operand; only
        # for >= 512 row tiles per launch (config 2: 2 x (524288 x 64 x 64)
        # 0.300 -> 0.244 ms; 2 x 16384 rows: 0.037 -> 0.046 ms, so not there)
        kin, ra, sra, ko, sko, rb, srb = view
        with _timed("gemm", 8 * nbat * m * n * k, 8 * (nbat * (m * k + k * n + m * n)),
                    detail + " V" if _timer else ""):
            for e in range(nbat):
                st = lib.qf_cgemm_c64_view(
                    _gemm_mode, 1, m, n, k, ctypes.c_void_p(big.data.data_ptr()), m * k, kin, ra,
                    sra, ko, sko, rb, srb, ctypes.c_void_p(B.data.data_ptr() + 8 * e * k * n),
                    max(n, 1), k * n, _lib.OP_N, ctypes.c_void_p(0), 0,
                    ctypes.c_void_p(out.data_ptr() + 8 * e * m * n), max(n, 1), m * n,
                    1.0, 0.0, 0.0, 0.0, stream_handle())
                if st != _lib.QF_OK:
                    break
        if st == _lib.QF_ERR_UNSUPPORTED and e == 0:
            st = None          # not describable after all: the paths below
    if st is not None:
        pass
    elif m <= 2 ** 22 and list(big.labels) != a_free + k_order:
        # big operand read in place through offset tables, broadcast over the batch
        roff, coff, rows_unit = _gather_tables(big.dims, big.labels, a_free, k_order,
                                               big.data.device)
        zeros = _zero_offsets(nbat, big.data.device)
        flags = _lib.GATHER_ROWS_UNIT if rows_unit else 0
        with _timed("gemm", 8 * nbat * m * n * k, 8 * (m * k + nbat * (k * n + m * n)), detail):
            st = lib.qf_cgemm_c64_gather_boff(
                _gemm_mode | flags, nbat, m, n, k, ctypes.c_void_p(big.data.data_ptr()),
                ctypes.c_void_p(zeros.data_ptr()), ctypes.c_void_p(roff.data_ptr()),
                ctypes.c_void_p(coff.data_ptr()), ctypes.c_void_p(B.data.data_ptr()), max(n, 1),
                k * n, _lib.OP_N, ctypes.c_void_p(out.data_ptr()), max(n, 1), m * n,
                1.0, 0.0, 0.0, 0.0, stream_handle())
    elif _row_blocks(big, a_free, k_order, n) is not None:
        # [outer rows][k][inner rows]: read in place in row blocks, no permute
        rin = _row_blocks(big, a_free, k_order, n)
        with _timed("gemm", 8 * nbat * m * n * k, 8 * (m * k + nbat * (k * n + m * n)),
                    detail + " R" if _timer else ""):
            st = lib.qf_cgemm_c64_rowblocks(
                _gemm_mode, nbat, m, n, k, ctypes.c_void_p(big.data.data_ptr()), rin, rin * k, rin,
                0, ctypes.c_void_p(B.data.data_ptr()), max(n, 1), k * n, _lib.OP_N,
                ctypes.c_void_p(out.data_ptr()), max(n, 1), m * n, 1.0, 0.0, 0.0, 0.0,
                stream_handle())
    else:
        # (too many rows for offset tables) one permute, then batch stride 0
        A = big.transpose_to(tuple(a_free + k_order))
        with _timed("gemm", 8 * nbat * m * n * k, 8 * (m * k + nbat * (k * n + m * n)), detail):
            st = lib.qf_cgemm_c64(_gemm_mode, nbat, m, n, k, ctypes.c_void_p(A.data.data_ptr()),
                                  max(k, 1), 0, _lib.OP_N, ctypes.c_void_p(B.data.data_ptr()),
                                  max(n, 1), k * n, _lib.OP_N, ctypes.c_void_p(out.data_ptr()),
                                  max(n, 1), m * n, 1.0, 0.0, 0.0, 0.0, stream_handle())
    _lib.check(st, "gemm_open")
    labels = tuple(so + a_free + s_free)
    dims = tuple(small.dim_of(l) for l in so) + tuple(big.dim_of(l) for l in a_free) + \
        tuple(small.dim_of(l) for l in s_free)
    return Tensor(labels, out, dims)


PATH_LABEL = "@p"


def _path_offsets(off, rep: int, stride: int):
    """Per-(bit-string, path value) entry bases: off[b] + j*stride, j fastest."""
    n = int(off.numel()) * rep
    out = torch.empty(max(n, 1), dtype=torch.int64, device=off.device)
    affine_offsets(out, n, rep, 0, base=off, stride=stride)
    return out[:n]


class ShapeOnly:
    """Labels and dims of a tensor that is never materialised (the fused
    intermediate of contract_late_expand), for flop/memory accounting."""
    __slots__ = ("labels", "dims", "itemsize")

    def __init__(self, labels, dims, itemsize: int = 8):
        self.labels, self.dims, self.itemsize = tuple(labels), tuple(dims), itemsize

    @property
    def nbytes(self) -> int:
        return math.prod(self.dims) * self.itemsize


_expand_enabled = True


def set_expand(enabled: bool) -> bool:
    """Enable/disable the re-associated (acc . op) . op2 of expand_plan; returns the previous value."""
    global _expand_enabled
    prev, _expand_enabled = _expand_enabled, bool(enabled)
    return prev


def expand_plan(acc: Tensor, op: Tensor, op2: Tensor, late: "LateBits", tail2=()):
    """Whether (acc . op) . op2 runs re-associated as acc . (op . op2): acc
    batched [@b][rb][ko][j] (j = the labels shared with op, innermost; ko =
    the labels op2 sums, right before j), op and op2 sites with open outputs
    sharing only ki.  The reference contracts acc with op first, widening
    each bit-string's 2^18-entry intermediate by op's free labels before op2
    sums them away again; op . op2 is tiny (one block per combination of the
    two sites' open outputs), and acc . (op . op2) is ONE batched GEMM
    [rb] x [(ko, j)] x [(ra, w_free)] per bit-string with the right block
    picked per entry (b_boff / b_nslice) -- the wide intermediate is never
    written.  Returns the plan dict or None."""
    if (late is None or not _expand_enabled or acc.buf.dtype != torch.complex64
            or op.buf.dtype != torch.complex64 or op2.buf.dtype != torch.complex64):
        return None
    lb = late.label
    bo, bo2 = late.outs(op), late.outs(op2)
    if not bo or not bo2 or lb in op.labels or lb in op2.labels:
        return None
    sliced = False
    if acc.labels and lb not in acc.labels and late.outs(acc):
        r = _expand_plan_open(acc, op, op2, late, tail2, bo, bo2)
        if r is not None:
            return r
        # an open operand the reference slices per bit-string: its slices
        # are the entries (TMA slice coordinates), like a batched operand
        ao = late.outs(acc)
        if (2 ** len(ao) <= late.limit or set(acc.labels[:len(ao)]) != set(ao)
                or acc._data is None):
            return None
        sliced = True
    elif not acc.labels or acc.labels[0] != lb or late.outs(acc) or acc._data is None:
        return None
    if any(_is_batch(l) for l in op.labels + op2.labels):
        return None
    lead = len(late.outs(acc)) if sliced else 1
    if any(_is_batch(l) for l in acc.labels[lead:]):
        return None
    core, cdims = list(acc.labels[lead:]), list(acc.dims[lead:])
    cset, oset, o2set = set(core), set(op.labels), set(op2.labels)
    j = [l for l in core if l in oset]
    ko = [l for l in core if l in o2set]
    if not j or not ko or set(j) & set(ko) or acc.size >= 2 ** 31:
        return None
    # A = acc's entries with k = its labels summed by op or op2 (memory
    # order): a plain row-major operand, or a TMA view of one
    k_order = [l for l in core if l in set(j) | set(ko)]
    rb = [l for l in core if l not in set(k_order)]
    view = None
    if core != rb + k_order:
        view = _a_view(core, cdims, rb, k_order)
        if view is None or _gemm_mode == _lib.GEMM_FFMA:
            return None
    ki = [l for l in op.labels if l in o2set]
    if not ki or any(l in cset for l in ki) or set(bo) & set(bo2):
        return None
    ra = [l for l in op.labels if l not in cset and l not in o2set and l not in bo]
    w_free = [l for l in op2.labels if l not in cset and l not in oset and l not in bo2]
    w_free = [l for l in w_free if l not in tail2] + [l for l in w_free if l in tail2]
    if not rb or not w_free:
        return None
    dim = dict(zip(acc.labels, acc.dims))
    dim.update(zip(op.labels, op.dims))
    dim.update(zip(op2.labels, op2.dims))
    P = lambda ls: math.prod(dim[l] for l in ls)
    M, K, N = P(rb), P(ko) * P(j), P(ra) * P(w_free)
    nb = late.nb if sliced else acc.dims[0]
    # the re-associated product must not cost more than the reference's two
    # contractions, and the per-combination blocks must stay small
    fused = M * K * N
    plain = M * P(ko) * P(j) * P(ra) * P(ki) + M * P(ra) * P(ko) * P(ki) * P(w_free)
    if fused > 1.25 * plain or 2 ** (len(bo) + len(bo2)) * K * N > 2 ** 22 or M < 128:
        return None
    u_lab = rb + ko + ra + ki
    u = ShapeOnly((lb,) + tuple(u_lab), (nb,) + tuple(dim[l] for l in u_lab))
    return {"j": j, "rb": rb, "ko": ko, "ra": ra, "ki": ki, "w_free": w_free, "bo": bo,
            "bo2": bo2, "M": M, "K": K, "N": N, "nb": nb, "u": u, "k_order": k_order,
            "view": view, "sliced": sliced,
            "labels": (lb,) + tuple(rb + ra + w_free),
            "dims": (nb,) + tuple(dim[l] for l in rb + ra + w_free)}


def _expand_plan_open(acc: Tensor, op: Tensor, op2: Tensor, late: "LateBits", tail2, bo, bo2):
    """expand_plan when acc still has open outputs (leading its layout): each
    bit-string's slice of acc is read in place as a TMA view at a slice
    coordinate (qf_cgemm_c64_view2), times its block of op . op2."""
    lb = late.label
    ao = late.outs(acc)
    if _gemm_mode == _lib.GEMM_FFMA:   # the view kernel is tensor-core only
        return None
    if (acc._data is None or set(acc.labels[:len(ao)]) != set(ao) or acc.size >= 2 ** 31
            or any(_is_batch(l) for l in acc.labels + op.labels + op2.labels)):
        return None
    core, cdims = list(acc.labels[len(ao):]), list(acc.dims[len(ao):])
    cset, oset, o2set = set(core), set(op.labels), set(op2.labels)
    j = [l for l in core if l in oset]
    ko = [l for l in core if l in o2set]
    ki = [l for l in op.labels if l in o2set]
    if not j or not ko or not ki or set(j) & set(ko) or any(l in cset for l in ki):
        return None
    if set(bo) & set(bo2) or set(ao) & (set(bo) | set(bo2)):
        return None
    k_order = [l for l in core if l in set(j) | set(ko)]
    rows = [l for l in core if l not in set(k_order)]
    view = _a_view(core, cdims, rows, k_order)
    if view is None or not rows:
        return None
    ra = [l for l in op.labels if l not in cset and l not in o2set and l not in bo]
    w_free = [l for l in op2.labels if l not in cset and l not in oset and l not in bo2]
    w_free = [l for l in w_free if l not in tail2] + [l for l in w_free if l in tail2]
    if not w_free:
        return None
    dim = dict(zip(acc.labels, acc.dims))
    dim.update(zip(op.labels, op.dims))
    dim.update(zip(op2.labels, op2.dims))
    P = lambda ls: math.prod(dim[l] for l in ls)
    M, K, N, nb = P(rows), P(k_order), P(ra) * P(w_free), late.nb
    # the reference order keeps acc . op open (once per output combination)
    # while that is cheaper than per bit-string; only fuse where the second
    # contraction would be sliced per bit-string anyway, and where the fused
    # per-bit-string product costs no more than both contractions
    comb1 = 2 ** (len(ao) + len(bo))
    if comb1 > late.limit or comb1 * 2 ** len(bo2) <= late.limit:
        return None
    fused = nb * M * K * N
    plain = comb1 * M * P(ko) * P(j) * P(ra) * P(ki) + nb * M * P(ra) * P(ko) * P(ki) * P(w_free)
    if (fused > 1.25 * plain or 2 ** (len(bo) + len(bo2)) * K * N > 2 ** 22 or M < 128
            or not 32 <= K <= 128):
        return None
    u_lab = ao + rows + ko + bo + ra + ki
    u = ShapeOnly(tuple(u_lab), tuple(dim[l] for l in u_lab))
    # every (acc slice, op/op2 output) combination at most as many as the
    # bit-strings: compute them all with the result's outputs kept open --
    # each acc slice read once (the op . op2 blocks side by side as column
    # blocks of one B) instead of once per bit-string
    keep = (2 ** (len(ao) + len(bo) + len(bo2)) <= nb and K <= 128
            and 2 ** (len(bo) + len(bo2)) * N <= 256)
    if keep:
        lab = ao + bo + bo2 + rows + ra + w_free
        return {"open": True, "keep_open": True, "view": view, "ao": ao, "k_order": k_order,
                "j": j, "rb": rows, "ko": ko, "ra": ra, "ki": ki, "w_free": w_free, "bo": bo,
                "bo2": bo2, "M": M, "K": K, "N": N, "nb": nb, "u": u, "labels": tuple(lab),
                "dims": tuple(dim[l] for l in lab)}
    return {"open": True, "view": view, "ao": ao, "k_order": k_order, "j": j, "rb": rows,
            "ko": ko, "ra": ra, "ki": ki, "w_free": w_free, "bo": bo, "bo2": bo2, "M": M,
            "K": K, "N": N, "nb": nb, "u": u, "labels": (lb,) + tuple(rows + ra + w_free),
            "dims": (nb,) + tuple(dim[l] for l in rows + ra + w_free)}


def contract_late_expand(acc: Tensor, op: Tensor, op2: Tensor, late: "LateBits", plan: dict):
    """Run an expand_plan: V = op . op2 (every open-output combination, a few
    blocks of [(ko, j)] x [(ra, w_free)]), then acc . V as one batched GEMM
    whose B block is chosen per bit-string (qf_cgemm_c64_ex2 b_boff /
    b_nslice: a TMA slice coordinate).  None if the library declines."""
    k_order = plan["k_order"]
    V = contract(op, op2)
    V = V.transpose_to(tuple(plan["bo"] + plan["bo2"] + k_order + plan["ra"] + plan["w_free"]))
    off = late.offsets(V, plan["bo"] + plan["bo2"])
    M, N, K, nb = plan["M"], plan["N"], plan["K"], plan["nb"]
    if plan.get("keep_open"):
        # all combinations: batch = acc's slices, B = every op . op2 block side
        # by side ([K][blocks x N]), C stored as [slice][block][M][N]
        nsl = 2 ** len(plan["ao"])
        nblk = 2 ** (len(plan["bo"]) + len(plan["bo2"]))
        V = V.transpose_to(tuple(k_order + plan["bo"] + plan["bo2"] + plan["ra"] +
                                 plan["w_free"]))
        entry = acc.size // nsl
        kin, ra, sra, ko, sko, rb, srb = plan["view"]
        out = device_buffer(nsl * nblk * M * N, acc.buf.dtype, acc.buf.device)
        zeros = _zero_offsets(nsl, acc.buf.device)
        NT = nblk * N
        with _timed("gemm", 8 * nsl * M * NT * K, 8 * nsl * (M * K + K * NT + M * NT),
                    f"b{nsl} m{M} n{NT} k{K} XK" if _timer else ""):
            st = _lib.load().qf_cgemm_c64_view2(
                _gemm_mode, nsl, M, NT, K, ctypes.c_void_p(acc.data.data_ptr()), entry,
                ctypes.c_void_p(0), 0, kin, ra, sra, ko, sko, rb, srb,
                ctypes.c_void_p(V.data.data_ptr()), NT, 0, _lib.OP_N,
                ctypes.c_void_p(zeros.data_ptr()), 1, ctypes.c_void_p(out.data_ptr()), N,
                nblk * M * N, N, M * N, 1.0, 0.0, 0.0, 0.0, stream_handle())
        if st == _lib.QF_ERR_UNSUPPORTED:
            return None
        _lib.check(st, "gemm_expand_keep")
        return Tensor(plan["labels"], out, plan["dims"])
    if plan.get("open"):
        # each bit-string's slice of acc read in place as a TMA view
        aoff = late.offsets(acc, plan["ao"])
        entry = acc.size // (2 ** len(plan["ao"]))
        kin, ra, sra, ko, sko, rb, srb = plan["view"]
        out = device_buffer(nb * M * N, acc.buf.dtype, acc.buf.device)
        with _timed("gemm", 8 * nb * M * N * K, 8 * nb * (M * K + K * N + M * N),
                    f"b{nb} m{M} n{N} k{K} XO" if _timer else ""):
            st = _lib.load().qf_cgemm_c64_view2(
                _gemm_mode, nb, M, N, K, ctypes.c_void_p(acc.data.data_ptr()), entry,
                ctypes.c_void_p(aoff.data_ptr()), 2 ** len(plan["ao"]), kin, ra, sra, ko, sko,
                rb, srb, ctypes.c_void_p(V.data.data_ptr()), max(N, 1), 0, _lib.OP_N,
                ctypes.c_void_p(off.data_ptr()), V.size // max(K * N, 1),
                ctypes.c_void_p(out.data_ptr()), max(N, 1), M * N, 0, 0, 1.0, 0.0, 0.0, 0.0,
                stream_handle())
        if st == _lib.QF_ERR_UNSUPPORTED:
            return None
        _lib.check(st, "gemm_expand_open")
        return Tensor(plan["labels"], out, plan["dims"])
    if plan.get("sliced"):
        # acc's per-bit-string slices (open outputs leading) as entries
        a_buf, a_off = acc.data, 0
        entry = acc.size // (2 ** len(late.outs(acc)))
        a_boff, a_nsl = late.offsets(acc, late.outs(acc)), 2 ** len(late.outs(acc))
    else:
        a_buf, a_off, entry = acc.raw()
        a_boff, a_nsl = None, 0
    vp = ctypes.c_void_p
    out = device_buffer(nb * M * N, acc.buf.dtype, acc.buf.device)
    if plan.get("view") is not None:
        # batched entries read as a TMA view (k split around a free run)
        kin, ra, sra, ko, sko, rb, srb = plan["view"]
        with _timed("gemm", 8 * nb * M * N * K, 8 * nb * (M * K + K * N + M * N),
                    f"b{nb} m{M} n{N} k{K} XV" if _timer else ""):
            st = _lib.load().qf_cgemm_c64_view2(
                _gemm_mode, nb, M, N, K, ctypes.c_void_p(a_buf.data_ptr() + 8 * a_off), entry,
                vp(a_boff.data_ptr() if a_boff is not None else 0), a_nsl, kin, ra, sra, ko,
                sko, rb, srb, ctypes.c_void_p(V.data.data_ptr()), max(N, 1), 0, _lib.OP_N,
                ctypes.c_void_p(off.data_ptr()), V.size // max(K * N, 1),
                ctypes.c_void_p(out.data_ptr()), max(N, 1), M * N, 0, 0, 1.0, 0.0, 0.0, 0.0,
                stream_handle())
        if st == _lib.QF_ERR_UNSUPPORTED:
            return None
        _lib.check(st, "gemm_expand_view")
        return Tensor(plan["labels"], out, plan["dims"])
    flags = _lib.BBOFF_EVEN if (K * N) % 2 == 0 else 0
    with _timed("gemm", 8 * nb * M * N * K, 8 * nb * (M * K + K * N + M * N),
                f"b{nb} m{M} n{N} k{K} X" if _timer else ""):
        st = _lib.load().qf_cgemm_c64_ex2(
            _gemm_mode | flags, nb, M, N, K, ctypes.c_void_p(a_buf.data_ptr() + 8 * a_off),
            max(K, 1), entry, _lib.OP_N, vp(a_boff.data_ptr() if a_boff is not None else 0),
            a_nsl, ctypes.c_void_p(0),
            ctypes.c_void_p(0), ctypes.c_void_p(V.data.data_ptr()), max(N, 1), 0, _lib.OP_N,
            ctypes.c_void_p(off.data_ptr()), V.size // max(K * N, 1),
            ctypes.c_void_p(out.data_ptr()), max(N, 1), M * N, 1.0, 0.0, 0.0, 0.0,
            stream_handle())
    if st == _lib.QF_ERR_UNSUPPORTED:
        return None
    _lib.check(st, "gemm_expand")
    return Tensor(plan["labels"], out, plan["dims"])


def contract_late_paths(a: Tensor, b: Tensor, late: LateBits, rep: int, tail=()) -> Optional[Tensor]:
    """contract_late inside a path-batched walk: batched operands carry
    nb*rep entries (bit-string major, path value fastest); an operand whose
    outputs are still open may carry the path value as a leading PATH_LABEL
    axis, and its per-(bit-string, value) slice is an entry base offset."""
    big, small = (a, b) if late._batched_size(a) >= late._batched_size(b) else (b, a)
    return _contract_sliced(big, small, late, tail, (), rep=rep)


def _contract_sliced(a: Tensor, b: Tensor, late: LateBits, tail=(), lead=(),
                     rep: int = 1) -> Optional[Tensor]:
    """One batched GEMM for a late-sliced network: `a` (the bigger operand)
    and `b` each either carry the batch axis or still have open outputs
    (b may also have neither -- broadcast).  An open operand's per-bit-string
    slice is an entry base offset (qf_cgemm_c64_ex a_boff / b_boff), so
    nothing is materialised: the big one is read in place (plain, through
    gathered tables, or as a cut-slice view), the small one is a site tensor
    with its outputs moved in front (memoised layout).  `lead`: kept-open cut
    labels; when they are all of b's free labels the result is stored
    transposed per entry ([@b, cut, rows]) so that per-path cut slices are
    contiguous (CUDA-core engines, N <= 16).  None if not eligible."""
    lb = late.label
    if a.buf.dtype != torch.complex64 or not _gather_enabled or a.size >= 2 ** 31:
        return None
    nb = late.nb * rep
    ao, bo = late.outs(a), late.outs(b)
    a_bat, b_bat = lb in a.labels, lb in b.labels
    if (a_bat and (ao or a.labels[0] != lb)) or (b_bat and bo) or (not a_bat and not ao):
        return None
    a_p, b_p = PATH_LABEL in a.labels, PATH_LABEL in b.labels
    if rep == 1 and (a_p or b_p):
        return None
    if (a_p and (not ao or a.labels[0] != PATH_LABEL)) or (b_p and (not bo or b.labels[0] != PATH_LABEL)):
        return None
    a_core = [l for l in a.labels if l != lb and l not in ao and l != PATH_LABEL]
    b_core = [l for l in b.labels if l != lb and l not in bo and l != PATH_LABEL]
    bset, aset = set(b_core), set(a_core)
    k_order = [l for l in a_core if l in bset]
    a_free = [l for l in a_core if l not in bset]
    b_free = [l for l in b_core if l not in aset]
    b_free = [l for l in b_free if l not in tail] + [l for l in b_free if l in tail]
    if any(_is_batch(l) for l in a_free + b_free):
        return None
    for l in k_order:
        if a.dim_of(l) != b.dim_of(l):
            raise ValueError(f"dimension mismatch on {l!r}: {a.dim_of(l)} vs {b.dim_of(l)}")
    m = math.prod(a.dim_of(l) for l in a_free)
    k = math.prod(a.dim_of(l) for l in k_order)
    n = math.prod(b.dim_of(l) for l in b_free)
    if k == 0 or k > 4096:
        return None
    lib = _lib.load()
    flags = 0
    # ---- A: batched entries (or a cut-slice view of them), or per-bit-string
    # slices of the open tensor
    a_boff = roff = coff = None
    if a_bat:
        a_buf, a_off, entry_a = a.raw()
    else:
        a_buf, a_off, entry_a = a.data, 0, 0
    if ao:
        st_a = _strides(a)
        if all(st_a[l] % 2 == 0 for l in ao + ([PATH_LABEL] if a_p else [])):
            flags |= _lib.BOFF_EVEN
    a_head = [PATH_LABEL] if a_p else []
    core_labels = a.labels[1:] if a_bat else tuple(l for l in a.labels
                                                   if l not in ao and l != PATH_LABEL)
    if list(core_labels) == a_free + k_order and (a_bat or list(a.labels) == a_head + ao + a_core):
        opA, lda = _lib.OP_N, max(k, 1)
    elif list(core_labels) == k_order + a_free and (a_bat or list(a.labels) == a_head + ao + a_core):
        opA, lda = _lib.OP_T, max(m, 1)
    else:
        if m > 2 ** 22:
            return None
        opA, lda, roff = _lib.OP_N, max(k, 1), "tables"
    if ao:
        a_boff = late.offsets(a, ao)
        if a_p:
            a_boff = _path_offsets(a_boff, rep, _strides(a)[PATH_LABEL])
        elif rep > 1:
            a_boff = _path_offsets(a_boff, rep, 0)
    # ---- B: batched entries, per-bit-string slices, or broadcast
    b_boff = None
    if bo:
        B = b.transpose_to(tuple(([PATH_LABEL] if b_p else []) + bo + k_order + b_free))
        opB, sB = _lib.OP_N, 0
        b_boff = late.offsets(B, bo)
        if b_p:
            b_boff = _path_offsets(b_boff, rep, _strides(B)[PATH_LABEL])
        elif rep > 1:
            b_boff = _path_offsets(b_boff, rep, 0)
        if all(_strides(B)[l] % 2 == 0 for l in bo + ([PATH_LABEL] if b_p else [])):
            flags |= _lib.BBOFF_EVEN
    elif b_bat:
        n_lay, t_lay = [lb] + k_order + b_free, [lb] + b_free + k_order
        if list(b.labels) == t_lay:
            B, opB = b, _lib.OP_T
        else:
            B, opB = b.transpose_to(tuple(n_lay)), _lib.OP_N
        sB = k * n
    else:
        B, opB, sB = b.transpose_to(tuple(k_order + b_free)), _lib.OP_N, 0
    ldb = max(n, 1) if opB == _lib.OP_N else max(k, 1)
    out = device_buffer(nb * m * n, a.buf.dtype, a.buf.device)
    labels_out = (lb,) + tuple(a_free) + tuple(b_free)
    dims = (nb,) + tuple(a.dim_of(l) for l in a_free) + tuple(b.dim_of(l) for l in b_free)
    c_trans = bool(lead) and bool(b_free) and set(b_free) <= set(lead) and n <= 16
    if c_trans:
        labels_out = (lb,) + tuple(b_free) + tuple(a_free)
        dims = (nb,) + tuple(b.dim_of(l) for l in b_free) + tuple(a.dim_of(l) for l in a_free)
    if roff == "tables" and a_bat and 32 <= k <= 128 and _view_enabled and _tview_enabled \
            and _gemm_mode != _lib.GEMM_FFMA and entry_a % 2 == 0 and (bo or b_bat):
        # rows innermost: a transposed TMA view (narrow N too; the kept cut
        # stored transposed straight from the tensor-core epilogue)
        tv = _a_tview(a.labels[1:], a.dims[1:], a_free, k_order)
        if tv is not None:
            ra, rb, srb, kin, ski, ko, sko = tv
            with _timed("gemm", 8 * nb * m * n * k, 8 * nb * (m * k + k * n + m * n),
                        f"b{nb} m{m} n{n} k{k} TV{'^T' if c_trans else ''}" if _timer else ""):
                st = _lib.load().qf_cgemm_c64_tview(
                    _gemm_mode | (_lib.C_TRANS if c_trans else 0), nb, m, n, k,
                    ctypes.c_void_p(a_buf.data_ptr() + 8 * a_off), entry_a, ra, rb, srb, kin, ski,
                    ko, sko, ctypes.c_void_p(B.data.data_ptr()), ldb, sB, opB,
                    ctypes.c_void_p(b_boff.data_ptr() if b_boff is not None else 0),
                    B.size // max(k * n, 1) if bo else 0, ctypes.c_void_p(out.data_ptr()),
                    max(m if c_trans else n, 1), m * n, 1.0, 0.0, 0.0, 0.0, stream_handle())
            if st != _lib.QF_ERR_UNSUPPORTED:
                _lib.check(st, "gemm_tview")
                return Tensor(labels_out, out, dims)
    if roff == "tables" and not c_trans:
        # batched big operand with scattered summed labels: a TMA-fed strided
        # view when it has one, else offset tables
        view = _a_view(a.labels[1:], a.dims[1:], a_free, k_order) if a_bat else None
        if view is not None and _gemm_view(
                nb, m, n, k, a_buf.data_ptr() + 8 * a_off, entry_a, view, B, ldb, sB, opB, out,
                b_boff, B.size // max(k * n, 1) if bo else 0):
            return Tensor(labels_out, out, dims)
    if roff == "tables":
        if a_bat:
            roff, coff, ru = _gather_tables(a.dims[1:], a.labels[1:], a_free, k_order,
                                            a.buf.device)
        else:
            roff, coff, ru = _gather_tables(a.dims, a.labels, a_free, k_order, a.buf.device)
        flags |= _lib.GATHER_ROWS_UNIT if ru else 0
    tag = ("G" if roff is not None else "NT"[opA]) + ("S" if ao else "") + \
        ("V" if a._data is None else "") + "," + ("S" if bo else "B" if b_bat else "0")
    if _timer is not None and os.environ.get("QF_DEBUG_LAYOUT"):
        tag += f" A{list(zip(a.labels, a.dims))} free{a_free} k{k_order} ao{ao} B{list(zip(b.labels, b.dims))} bfree{b_free} bo{bo}"
    vp = ctypes.c_void_p
    # site-tensor slices picked per entry are whole [K][N] blocks of B
    b_nslice = B.size // max(k * n, 1) if bo else 0

    def launch(trans: bool):
        with _timed("gemm", 8 * nb * m * n * k, 8 * nb * (m * k + k * n + m * n),
                    f"b{nb} m{m} n{n} k{k} {tag}{'^T' if trans else ''}" if _timer else ""):
            return lib.qf_cgemm_c64_ex2(
                _gemm_mode | flags | (_lib.C_TRANS if trans else 0), nb, m, n, k,
                vp(a_buf.data_ptr() + 8 * a_off), lda, entry_a, opA,
                vp(a_boff.data_ptr() if a_boff is not None else 0), 0,
                vp(roff.data_ptr() if roff is not None else 0),
                vp(coff.data_ptr() if coff is not None else 0),
                vp(B.data.data_ptr()), ldb, sB, opB,
                vp(b_boff.data_ptr() if b_boff is not None else 0), b_nslice,
                vp(out.data_ptr()), max(m if trans else n, 1), m * n, 1.0, 0.0, 0.0, 0.0,
                stream_handle())

    st = launch(c_trans)
    if c_trans and st == _lib.QF_ERR_UNSUPPORTED:    # row-major result after all
        labels_out = (lb,) + tuple(a_free) + tuple(b_free)
        dims = (nb,) + tuple(a.dim_of(l) for l in a_free) + tuple(b.dim_of(l) for l in b_free)
        st = launch(False)
    _lib.check(st, "gemm_ex")
    return Tensor(labels_out, out, dims)

# ---------------------------------------------------------------------------
# path batching: a cut's values as one more batch dimension


_BCAST: dict = {}


def _bcast_offsets(n: int, rep: int, entry: int, device):
    """int64 entry bases (e // rep) * entry, e < n: entry e of a path-batched
    walk reads entry e // rep of an operand that has no path index."""
    key = (n, rep, entry, str(device))
    hit = _BCAST.get(key)
    if hit is None:
        hit = torch.empty(max(n, 1), dtype=torch.int64, device=device)
        affine_offsets(hit, n, rep, entry)
        hit = hit[:n]
        if len(_BCAST) > 64:
            _BCAST.clear()
        _BCAST[key] = hit
    return hit


def contract_bcast(x: Tensor, y: Tensor, rep: int, tail=(), label: str = "@b") -> Optional[Tensor]:
    """Contract a path-batched operand `x` (leading `label` axis of nb*rep
    entries, path index fastest) with `y`, which has no path index (leading
    `label` axis of nb entries, or no batch axis at all): `y` is broadcast
    over the paths through per-entry base offsets (qf_cgemm_c64_ex a_boff /
    b_boff), nothing is copied.  Same products as `rep` separate
    contractions.  None when not expressible (caller falls back)."""
    if x.buf.dtype != torch.complex64 or y.buf.dtype != torch.complex64 or x.labels[0] != label:
        return None
    y_bat = bool(y.labels) and y.labels[0] == label
    NB = x.dims[0]
    nb = y.dims[0] if y_bat else 1
    if NB != nb * rep or any(_is_batch(l) for l in x.labels[1:] + y.labels[int(y_bat):]):
        return None
    xc, yc = list(x.labels[1:]), list(y.labels[int(y_bat):])
    xs, ys = set(xc), set(yc)
    y_entry = y.size // nb
    x_entry = x.size // NB
    big_is_x = x_entry >= y_entry
    a, b = (x, y) if big_is_x else (y, x)
    a_core, b_core = (xc, yc) if big_is_x else (yc, xc)
    bset, aset = (ys, xs) if big_is_x else (xs, ys)
    k_order = [l for l in a_core if l in bset]
    a_free = [l for l in a_core if l not in bset]
    b_free = [l for l in b_core if l not in aset]
    b_free = [l for l in b_free if l not in tail] + [l for l in b_free if l in tail]
    for l in k_order:
        if a.dim_of(l) != b.dim_of(l):
            raise ValueError(f"dimension mismatch on {l!r}: {a.dim_of(l)} vs {b.dim_of(l)}")
    m = math.prod(a.dim_of(l) for l in a_free)
    k = math.prod(a.dim_of(l) for l in k_order)
    n = math.prod(b.dim_of(l) for l in b_free)
    a_head = [label] if (big_is_x or y_bat) else []
    b_head = [label] if (not big_is_x or y_bat) else []
    if list(a.labels) == a_head + a_free + k_order:
        A, opA, lda = a, _lib.OP_N, max(k, 1)
    elif list(a.labels) == a_head + k_order + a_free:
        A, opA, lda = a, _lib.OP_T, max(m, 1)
    else:
        A, opA, lda = a.transpose_to(tuple(a_head + a_free + k_order)), _lib.OP_N, max(k, 1)
    if list(b.labels) == b_head + k_order + b_free:
        B, opB, ldb = b, _lib.OP_N, max(n, 1)
    elif list(b.labels) == b_head + b_free + k_order:
        B, opB, ldb = b, _lib.OP_T, max(k, 1)
    else:
        B, opB, ldb = b.transpose_to(tuple(b_head + k_order + b_free)), _lib.OP_N, max(n, 1)
    dev = x.buf.device
    flags = 0
    a_boff = b_boff = None
    if big_is_x:
        sA, sB = m * k, k * n
        b_boff = _bcast_offsets(NB, rep, k * n if y_bat else 0, dev)
        if (k * n) % 2 == 0 or not y_bat:
            flags |= _lib.BBOFF_EVEN
    else:
        sA, sB = m * k, k * n
        a_boff = _bcast_offsets(NB, rep, m * k if y_bat else 0, dev)
        if (m * k) % 2 == 0 or not y_bat:
            flags |= _lib.BOFF_EVEN
    out = device_buffer(NB * m * n, x.buf.dtype, dev)
    vp = ctypes.c_void_p
    with _timed("gemm", 8 * NB * m * n * k, 8 * (NB * m * n + (NB if big_is_x else nb) * m * k +
                                                  (nb if big_is_x else NB) * k * n),
                f"b{NB} m{m} n{n} k{k} P{rep}" if _timer else ""):
        st = _lib.load().qf_cgemm_c64_ex(
            _gemm_mode | flags, NB, m, n, k, vp(A.data.data_ptr()), lda, sA, opA,
            vp(a_boff.data_ptr() if a_boff is not None else 0), vp(0), vp(0),
            vp(B.data.data_ptr()), ldb, sB, opB,
            vp(b_boff.data_ptr() if b_boff is not None else 0),
            vp(out.data_ptr()), max(n, 1), m * n, 1.0, 0.0, 0.0, 0.0, stream_handle())
    _lib.check(st, "gemm_bcast")
    labels = (label,) + tuple(a_free) + tuple(b_free)
    dims = (NB,) + tuple(a.dim_of(l) for l in a_free) + tuple(b.dim_of(l) for l in b_free)
    return Tensor(labels, out, dims)


_ONES: dict = {}


def sum_path_axis(t: Tensor, rep: int, keep_batch: bool, label: str = "@b") -> Tensor:
    """Sum a path-batched tensor (leading `label` axis of nb*rep entries,
    path index fastest) over its path index: one batched GEMM with a ones
    row, C[b] (1 x R) = 1 (1 x rep) @ t[b] (rep x R).  keep_batch=False
    drops the (then size-1) batch axis."""
    NB = t.dims[0]
    nb = NB // rep
    R = t.size // NB
    key = (rep, str(t.buf.dtype), str(t.buf.device))
    ones = _ONES.get(key)
    if ones is None:
        ones = _ONES[key] = torch.empty(rep, dtype=t.buf.dtype, device=t.buf.device)
        st = _lib.load().qf_fill_value(ctypes.c_void_p(ones.data_ptr()), rep, 1.0, 0.0,
                                       _elem_bytes(ones), stream_handle())
        _lib.check(st, "fill_value")
    out = device_buffer(nb * R, t.buf.dtype, t.buf.device)
    lib = _lib.load()
    with _timed("gemm", 8 * nb * R * rep, _elem_bytes(out) * (NB * R + nb * R),
                f"b{nb} m1 n{R} k{rep} sum" if _timer else ""):
        st = _gemm_call(lib, nb, 1, R, rep, ones, rep, _lib.OP_N, t.data, R, _lib.OP_N, out, 0,
                        rep * R, R, 1.0, 0.0, None)
    _lib.check(st, "sum_paths")
    if keep_batch:
        return Tensor(t.labels, out, (nb,) + t.dims[1:])
    return Tensor(t.labels[1:], out, t.dims[1:])


# ---------------------------------------------------------------------------
# permutation API shims (reference signatures; one device pass whatever the plan)


@dataclass(frozen=True)
class Move:
    """One pass of the reference's CPU decomposition (rq/tensor_core.py:41-57):
    an "L" move permutes the leading axes and leaves the trailing `gamma`
    axes in place, an "R" move permutes the trailing `gamma` axes;
    `group_perm` is in gather order over the affected group."""

    kind: str
    group_perm: tuple
    gamma: int

    def __post_init__(self):
        if self.kind not in ("L", "R"):
            raise ValueError(f"move kind must be 'L' or 'R', got {self.kind!r}")


@dataclass(frozen=True)
class PermutePlan:
    """(dims, perm) of a transpose plus the reference's L/R move list.

    The reference executes `moves` as cache-sized CPU passes
    (rq/tensor_core.py:81-206).  On the B200 the whole permutation is ONE
    shared-memory-tiled pass (K1) whatever the moves say: they are kept as
    plan metadata with the reference's decomposition rules so that callers
    inspecting `move_summary()` / `fallback` see the same plan, and
    `device_pass` names what actually runs."""

    dims: tuple
    perm: tuple
    moves: tuple = ()
    mu: int = 5
    nu: int = 10
    fallback: Optional[str] = None
    device_pass: str = "tiled"

    @property
    def out_dims(self) -> tuple:
        return tuple(self.dims[p] for p in self.perm)

    def move_summary(self) -> list:
        return [(m.kind, m.gamma) for m in self.moves]


def _in_place(seq) -> bool:
    return all(v == i for i, v in enumerate(seq))


def _vol(dims, axes) -> int:
    return math.prod(dims[a] for a in axes)


def _moves_three(dims, perm, lo: int, hi: int):
    """The general L-R-L template (rq/tensor_core.py:154-206): a left move
    parks the axes that must end up trailing next to the window, a right
    move orders the final suffix, a last left move orders the prefix.
    Returns the move tuple or None when no (gamma_L, gamma_R) fits."""
    k = len(dims)
    rank_of = {a: j for j, a in enumerate(perm)}
    # smallest suffix length whose input AND output blocks reach the L bound
    g_l = next((g for g in range(1, k)
                if _vol(dims, range(k - g, k)) >= lo and _vol(dims, perm[k - g:]) >= lo), None)
    if g_l is None:
        return None
    head = k - g_l
    tail_axes = list(perm[head:])
    strays = [a for a in tail_axes if a < head]           # must cross into the suffix
    stay = sorted((a for a in range(head) if a not in tail_axes), key=rank_of.__getitem__)
    first = stay + strays
    lay = first + list(range(head, k))
    # widest R window within the budget that still covers strays + suffix
    need = g_l + len(strays)
    g_r = next((g for g in range(k, need - 1, -1) if _vol(dims, lay[k - g:]) <= hi), None)
    if g_r is None:
        return None
    moves = []
    if not _in_place(first):
        moves.append(Move("L", tuple(first), g_l))
    win = lay[k - g_r:]
    rest = sorted((a for a in win if a not in tail_axes), key=rank_of.__getitem__)
    target = rest + tail_axes
    local = tuple(win.index(a) for a in target)
    if not _in_place(local):
        moves.append(Move("R", local, g_r))
    lay = lay[:k - g_r] + target
    now = lay[:head]
    last = tuple(now.index(a) for a in perm[:head])
    if not _in_place(last):
        moves.append(Move("L", last, g_l))
    return tuple(moves)


def _plan_moves(dims, perm, mu: int, nu: int):
    """(moves, fallback) by the reference's rules, tried in its order:
    identity; fixed suffix of >= 2^mu entries -> one L; fixed prefix with a
    window of <= 2^nu entries -> one R; a prefix block mapped onto itself
    with the rest a legal window -> L then R; the L-R-L template; else the
    naive fallback (rq/tensor_core.py:81-151)."""
    k = len(dims)
    lo, hi = 1 << mu, 1 << nu
    if _in_place(perm):
        return (), None
    fixed_tail = next((g for g in range(k + 1) if g == k or perm[k - 1 - g] != k - 1 - g), k)
    if fixed_tail >= 1 and _vol(dims, range(k - fixed_tail, k)) >= lo:
        return (Move("L", tuple(perm[:k - fixed_tail]), fixed_tail),), None
    fixed_head = next((g for g in range(k + 1) if g == k or perm[g] != g), k)
    if _vol(dims, range(fixed_head, k)) <= hi:
        return (Move("R", tuple(p - fixed_head for p in perm[fixed_head:]), k - fixed_head),), None
    # largest b with perm[:b] a permutation of 0..b-1 and a legal trailing window
    split, top = None, -1
    for b in range(1, k):
        top = max(top, perm[b - 1])
        if top == b - 1 and lo <= _vol(dims, range(b, k)) <= hi:
            split = b
    if split is not None:
        out = []
        if not _in_place(perm[:split]):
            out.append(Move("L", tuple(perm[:split]), k - split))
        back = tuple(p - split for p in perm[split:])
        if not _in_place(back):
            out.append(Move("R", back, k - split))
        return tuple(out), None
    three = _moves_three(dims, perm, lo, hi)
    if three is not None:
        return three, None
    return (), "naive"


def moves_compose(plan: "PermutePlan") -> tuple:
    """The permutation obtained by applying `plan.moves` in order (gather
    order, like `perm`) -- equals plan.perm unless the plan fell back."""
    k = len(plan.dims)
    lay = list(range(k))
    for m in plan.moves:
        if m.kind == "L":
            head = lay[:k - m.gamma]
            lay = [head[j] for j in m.group_perm] + lay[k - m.gamma:]
        else:
            win = lay[k - m.gamma:]
            lay = lay[:k - m.gamma] + [win[j] for j in m.group_perm]
    return tuple(lay)


def plan_permutation(dims: Sequence[int], perm: Sequence[int], mu: int = 5, nu: int = 10) -> PermutePlan:
    dims = tuple(int(d) for d in dims)
    perm = tuple(int(p) for p in perm)
    if sorted(perm) != list(range(len(dims))):
        raise ValueError(f"perm {perm} is not a permutation of 0..{len(dims) - 1}")
    if mu < 0 or nu < mu:
        raise ValueError(f"need 0 <= mu <= nu, got mu={mu}, nu={nu}")
    if any(d < 1 for d in dims):
        raise ValueError("dims must be positive")
    moves, fallback = _plan_moves(dims, perm, mu, nu)
    return PermutePlan(dims, perm, moves, mu, nu, fallback,
                       "none" if _in_place(perm) else "tiled")


def _as_device(array):
    if torch is not None and isinstance(array, torch.Tensor):
        return array.reshape(-1), None
    arr = np.ascontiguousarray(array)
    if arr.dtype not in _TORCH_OF:
        # K1 moves 8- and 16-byte elements without touching their bits: other
        # 8/16-byte dtypes (float64, int64, ...) ride through as raw elements
        if arr.dtype.itemsize not in (8, 16) or arr.dtype.hasobject:
            raise ValueError("permutation supports 8- and 16-byte elements "
                             f"(complex64/complex128, float64, int64), got {arr.dtype}")
        raw = arr.reshape(-1).view(np.complex64 if arr.dtype.itemsize == 8 else np.complex128)
        _require_cuda()
        return torch.from_numpy(raw).to(torch.cuda.current_device()), arr.dtype
    _require_cuda()
    return torch.from_numpy(arr.reshape(-1)).to(torch.cuda.current_device()), arr.dtype


def permute_fast(array, plan: PermutePlan, thread_count: int = 1, workspace=None, map_cache=None):
    """Apply `plan` on the device.  numpy in -> numpy out; torch in -> torch out."""
    data, np_dtype = _as_device(array)
    out = permute_buffer(data, plan.dims, plan.perm)[: math.prod(plan.dims)]
    if np_dtype is None:
        return out.view(plan.out_dims) if len(plan.out_dims) <= 25 else out
    return out.cpu().numpy().view(np_dtype).reshape(plan.out_dims)


def permute_naive(array, perm: Sequence[int]):
    """Same result as the reference's numpy transpose, computed by K1."""
    shape = tuple(array.shape)
    return permute_fast(array, plan_permutation(shape, perm))


# ---------------------------------------------------------------------------
# permutation micro-benchmark (reference: rq/tensor_core.py:427-511)


def _random_perm(rng, k: int, fix_prefix: int = 0, fix_suffix: int = 0) -> tuple:
    """Random non-identity permutation fixing the given prefix/suffix
    (same draw sequence as the reference's benchmark)."""
    body = list(range(fix_prefix, k - fix_suffix))
    while True:
        mixed = [int(v) for v in rng.permutation(body)]
        if mixed != body:
            return tuple(range(fix_prefix)) + tuple(mixed) + tuple(range(k - fix_suffix, k))


def benchmark_permute(rank: int = 20, gammas=range(5, 11), thread_counts=(1,), repeats: int = 7,
                      dtype=np.complex64, compare_backends: bool = False, seed: int = 0) -> list:
    """Device-timed twin of the reference's benchmark_permute: per gamma an
    "L move" (leading axes permuted, trailing gamma fixed), an "R move"
    (trailing gamma permuted) and a "naive" full permutation of a binary
    rank-`rank` tensor, with the same seeded permutations.  Rows keep the
    reference schema (op, rank, gamma, threads, median_ns, p10_ns, p90_ns);
    every op is one K1 launch, timed with CUDA events after a warm-up, and
    `threads` is echoed only for schema compatibility."""
    _require_cuda()
    rng = np.random.Generator(np.random.PCG64(seed))
    x = (rng.standard_normal(1 << rank) + 1j * rng.standard_normal(1 << rank)).astype(dtype)
    src = torch.from_numpy(x).cuda()
    dst = torch.empty_like(src)
    dims = (2,) * rank

    def time_ns(perm):
        permute_buffer(src, dims, perm, out=dst)  # warm: plan + tables
        samples = []
        for _ in range(repeats):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            permute_buffer(src, dims, perm, out=dst)
            b.record()
            torch.cuda.synchronize()
            samples.append(a.elapsed_time(b) * 1e6)
        arr = np.array(samples)
        return float(np.median(arr)), float(np.percentile(arr, 10)), float(np.percentile(arr, 90))

    rows = []
    for gamma in gammas:
        perm_l = _random_perm(rng, rank, fix_suffix=gamma)
        perm_r = _random_perm(rng, rank, fix_prefix=rank - gamma)
        for name, perm in (("lmove", perm_l), ("rmove", perm_r)):
            med, p10, p90 = time_ns(perm)
            for threads in thread_counts:
                op = f"{name}/b200" if compare_backends else name
                rows.append({"op": op, "rank": rank, "gamma": gamma, "threads": threads,
                             "median_ns": med, "p10_ns": p10, "p90_ns": p90})
        perm_full = _random_perm(rng, rank)
        med, p10, p90 = time_ns(perm_full)
        rows.append({"op": "naive", "rank": rank, "gamma": gamma, "threads": 1,
                     "median_ns": med, "p10_ns": p10, "p90_ns": p90})
    return rows


def benchmark_csv(rows: list) -> str:
    header = ["op", "rank", "gamma", "threads", "median_ns", "p10_ns", "p90_ns"]
    return "\n".join([",".join(header)] + [",".join(str(r[h]) for h in header) for r in rows]) + "\n"
