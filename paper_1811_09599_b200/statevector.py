"""Dense state-vector simulation on the B200 (complex128) for verification.

The B200 twin of the reference's verification simulator `rqcsim.oracle`
(rq/oracle.py:51-92: evolve, exact_amplitude, exact_distribution; kernels
rq/_kernels.py:162-271).  It is independent of the tensor-network path --
gates are applied cycle by cycle to the full 2^n state -- and exists to
cross-check that path's amplitudes exactly where the host simulator cannot
(the reference caps it at 26 qubits; 2^33 complex128 amplitudes are 128 GiB
of the 180 GB HBM).

Each cycle's gates act on disjoint qubits (they commute), so they are
packed into a few passes; a pass stages tiles of 2^k amplitudes over k <= 10
chosen bits (the 5 lowest always among them, so every warp touches 512
contiguous bytes) in shared memory and applies all of its gates there
(`qf_sv_apply`, csrc/qf_statevec.cu).  Conventions follow the reference:
qubit 0 is the most significant bit of the state index (rq/oracle.py:8-10).
"""

from __future__ import annotations

import ctypes
from typing import Sequence, Union

import numpy as np

from . import _lib
from .circuits import Circuit
from .network_builder import _ONE_Q
from .tensor_core import _require_cuda, stream_handle, torch

MAX_QUBITS = 33
TILE_BITS = 10
LOW_BITS = 5
MAX_OPS = 24
_KIND = {"cz": 1, "iswap": 2}


def bits_to_index(bits: str) -> int:
    """Bit-string (leftmost char = qubit 0) to state index (rq/oracle.py:41-43)."""
    return int(bits, 2)


def index_to_bits(index: int, n: int) -> str:
    return format(index, f"0{n}b")


def _check_size(circuit: Circuit):
    if circuit.n > MAX_QUBITS:
        raise ValueError(f"GPU state vector capped at {MAX_QUBITS} qubits, got {circuit.n}")


def plan_passes(gates: Sequence, n: int, tile_bits: int = TILE_BITS) -> list:
    """Pack one cycle's gates (disjoint qubits) into passes: each pass is
    (ascending tile bit positions, [gate, ...]) with the LOW_BITS lowest bits
    always in the tile and every gate's bits inside it."""
    k = min(tile_bits, n)
    low = set(range(min(LOW_BITS, n)))
    passes, cur_bits, cur = [], set(low), []
    for g in gates:
        gb = {n - 1 - q for q in g.qubits}
        if len(cur_bits | gb) > k or len(cur) == MAX_OPS:
            passes.append((cur_bits, cur))
            cur_bits, cur = set(low), []
        cur_bits |= gb
        cur.append(g)
    if cur:
        passes.append((cur_bits, cur))
    out = []
    for bits, gs in passes:
        # fill the tile up to k bits with the lowest unused positions (whole tiles)
        extra = [p for p in range(n) if p not in bits]
        bits = sorted(bits | set(extra[:k - len(bits)]))
        out.append((bits, gs))
    return out


def _apply_pass(psi, n: int, bits: list, gates: list):
    pos = {b: j for j, b in enumerate(bits)}
    kinds, obits, mats = [], [], []
    for g in gates:
        if len(g.qubits) == 1:
            m = _ONE_Q[g.name]
            kinds.append(0)
            obits += [pos[n - 1 - g.qubits[0]], 0]
            mats += [m[0, 0].real, m[0, 0].imag, m[0, 1].real, m[0, 1].imag,
                     m[1, 0].real, m[1, 0].imag, m[1, 1].real, m[1, 1].imag]
        else:
            if g.name not in _KIND:
                raise ValueError(f"unsupported two-qubit gate {g.name!r}")
            a, b = g.qubits
            kinds.append(_KIND[g.name])
            obits += [pos[n - 1 - a], pos[n - 1 - b]]
            mats += [0.0] * 8
    i32, f64 = ctypes.c_int32, ctypes.c_double
    st = _lib.load().qf_sv_apply(
        ctypes.c_void_p(psi.data_ptr()), n, len(bits), (i32 * len(bits))(*bits), len(gates),
        (i32 * max(1, len(kinds)))(*kinds), (i32 * max(2, len(obits)))(*obits),
        (f64 * max(8, len(mats)))(*mats), stream_handle())
    _lib.check(st, "sv_apply")


def evolve_device(circuit: Circuit, in_bits: Union[str, int] = 0):
    """Output state |psi> = U|in> as a flat complex128 device tensor."""
    _check_size(circuit)
    _require_cuda()
    n = circuit.n
    psi = torch.empty(1 << n, dtype=torch.complex128, device=torch.cuda.current_device())
    idx = bits_to_index(in_bits) if isinstance(in_bits, str) else int(in_bits)
    _lib.check(_lib.load().qf_sv_basis(ctypes.c_void_p(psi.data_ptr()), n, idx, stream_handle()),
               "sv_basis")
    for gates in circuit.by_cycle():
        for bits, gs in plan_passes(gates, n):
            _apply_pass(psi, n, bits, gs)
    return psi


def evolve(circuit: Circuit, in_bits: Union[str, int] = 0) -> np.ndarray:
    """Full output state vector (host copy; rq/oracle.py:51-74)."""
    return evolve_device(circuit, in_bits).cpu().numpy()


def exact_amplitudes(circuit: Circuit, in_bits: Union[str, int], out_bits: Sequence,
                     psi=None) -> np.ndarray:
    """<out|U|in> for many bit-strings (one device gather)."""
    if psi is None:
        psi = evolve_device(circuit, in_bits)
    idx = np.array([bits_to_index(b) if isinstance(b, str) else int(b) for b in out_bits],
                   dtype=np.int64)
    if idx.size == 0:
        return np.zeros(0, dtype=np.complex128)
    if idx.min() < 0 or idx.max() >= psi.numel():
        raise ValueError("bit-string index out of range")
    d_idx = torch.from_numpy(idx).to(psi.device)
    out = torch.empty(idx.size, dtype=torch.complex128, device=psi.device)
    st = _lib.load().qf_sv_gather(ctypes.c_void_p(psi.data_ptr()), ctypes.c_void_p(d_idx.data_ptr()),
                                  int(idx.size), ctypes.c_void_p(out.data_ptr()), stream_handle())
    _lib.check(st, "sv_gather")
    return out.cpu().numpy()


def exact_amplitude(circuit: Circuit, in_bits: Union[str, int], out_bits: Union[str, int]) -> complex:
    return complex(exact_amplitudes(circuit, in_bits, [out_bits])[0])


def exact_distribution(circuit: Circuit, in_bits: Union[str, int] = 0) -> np.ndarray:
    """|<b|U|in>|^2 for all 2^n bit-strings (rq/oracle.py:84-92)."""
    psi = evolve_device(circuit, in_bits)
    return (psi.real ** 2 + psi.imag ** 2).cpu().numpy()
