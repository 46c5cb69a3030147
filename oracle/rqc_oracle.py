"""CPU oracle for the RQC amplitude path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(`rqcsim`, /root/reference/pkg/src/rqcsim) for the hot path that the
B200 package accelerates.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import it, and
only as the checker or the timed CPU baseline.  The product package
(`paper_1811_09599_b200`) never imports, links or calls anything here.

Parity pin: every function below is checked against golden vectors that
`tests/golden/make_golden.py` produced by importing the reference itself
(circuit text, plan text, amplitudes, batch amplitudes, PathStats flops,
permutation bytes).  See tests/test_oracle_golden.py.

Inputs are the reference's own text formats (circuit file, plan file),
so the oracle does not depend on the product's host code either.

Reference map (rq/ = pkg/src/rqcsim/):
  lattice geometry            rq/circuits.py:48-152   (edges 68-78)
  circuit text format         rq/circuits.py:417-488
  gate matrices / CZ factors  rq/network_builder.py:30-58
  per-site time contraction   rq/network_builder.py:152-256 (build_3d + contract_time)
  bond merge order            rq/network_builder.py:239-253, 259-289
  plan text + analysis        rq/contraction_plan.py:155-328
  path enumeration            rq/contraction_plan.py:359-405
  executor (reuse cache)      rq/contraction_plan.py:450-523
  pairwise contraction        rq/tensor_core.py:391-419
  permutation oracle          rq/tensor_core.py:271-273
  amplitude / batch           rq/amplitude_engine.py:114-170
"""

from __future__ import annotations

import itertools
import math
import re
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

# ---------------------------------------------------------------------------
# permutation oracle (rq/tensor_core.py:271-273)


def permute_naive(array: np.ndarray, perm: Sequence[int]) -> np.ndarray:
    """numpy strided transpose into fresh row-major storage (bit-exact oracle)."""
    return np.ascontiguousarray(np.transpose(array, tuple(perm)))


# ---------------------------------------------------------------------------
# lattices (rq/circuits.py:48-152)


def lattice_sites(kind: str) -> list[tuple[int, int]]:
    """Row-major sorted (row, col) sites for `grid:RxC` and the diamond
    bristlecone-70/72 frames (the reference ships these as coordinate
    tables; the diamond is regenerated here from its closed form)."""
    kind = kind.strip().lower()
    m = re.fullmatch(r"grid:(\d+)x(\d+)", kind)
    if m:
        r, c = int(m.group(1)), int(m.group(2))
        return [(i, j) for i in range(r) for j in range(c)]
    if kind == "bristlecone-70":
        out = []
        for r in range(10):
            h = r if r < 5 else 9 - r
            out.extend((r, c) for c in range(4 - h, 7 + h))
        return out
    if kind == "bristlecone-72":
        out = [(0, 5)]
        out.extend((r + 1, c) for r, c in lattice_sites("bristlecone-70"))
        out.append((11, 5))
        return out
    m = re.fullmatch(r"bristlecone-(\d+)", kind)
    if m:   # the reference's coordinate tables, as its own golden fixture holds them
        import json
        import os
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "tests", "golden", "golden_shipped.json")
        with open(path) as fh:
            table = json.load(fh)["lattices"].get(m.group(1))
        if table is not None:
            return sorted(tuple(x) for x in table["sites"])
    raise ValueError(f"oracle has no lattice {kind!r}")


def lattice_edges(sites: Sequence[tuple[int, int]]) -> list[tuple[int, int]]:
    """(low id, high id) pairs; right neighbour before down neighbour, per
    site in id order (rq/circuits.py:68-78)."""
    index = {rc: i for i, rc in enumerate(sites)}
    edges = []
    for i, (r, c) in enumerate(sites):
        for dr, dc in ((0, 1), (1, 0)):
            j = index.get((r + dr, c + dc))
            if j is not None:
                edges.append((i, j))
    return edges


# ---------------------------------------------------------------------------
# circuit text (rq/circuits.py:393-488)


@dataclass
class OracleCircuit:
    n: int
    lattice: str
    t: int
    gates: list  # (cycle, name, qubits)
    sites: list = field(default_factory=list)
    edges: list = field(default_factory=list)


def parse_circuit(text: str) -> OracleCircuit:
    lines = text.splitlines()
    n = int(lines[0].strip())
    meta = {}
    gates = []
    max_cycle = 0
    for raw in lines[1:]:
        s = raw.strip()
        if not s:
            continue
        if s.startswith("#"):
            m = re.fullmatch(r"#\s*(\w+)\s*:\s*(.+?)\s*", s)
            if m:
                meta[m.group(1)] = m.group(2)
            continue
        parts = s.split()
        cyc = int(parts[0])
        gates.append((cyc, parts[1].lower(), tuple(int(p) for p in parts[2:])))
        max_cycle = max(max_cycle, cyc)
    kind = meta["lattice"]
    if "depth" in meta:
        t = int(re.fullmatch(r"1\+(\d+)\+1", meta["depth"]).group(1))
    else:
        t = max(0, max_cycle - 1)
    sites = lattice_sites(kind)
    if len(sites) != n:
        raise ValueError("qubit count does not match lattice")
    gates.sort(key=lambda g: (g[0], g[2]))
    return OracleCircuit(n, kind, t, gates, sites, lattice_edges(sites))


# ---------------------------------------------------------------------------
# gates (rq/network_builder.py:28-58); U[out, in]

_H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2.0)
_T = np.diag([1.0, np.exp(1j * np.pi / 4)]).astype(np.complex128)
_SX = 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]], dtype=np.complex128)
_SY = 0.5 * np.array([[1 + 1j, -1 - 1j], [1 + 1j, 1 + 1j]], dtype=np.complex128)
ONE_Q = {"h": _H, "t": _T, "x_1_2": _SX, "y_1_2": _SY}


def _two_qubit_factors():
    # g[bond, in, out]; sum_b ga[b,i1,o1] gb[b,i2,o2] = <o1 o2|U|i1 i2>
    cz_a = np.zeros((2, 2, 2), np.complex128)
    cz_a[0, 0, 0] = cz_a[1, 1, 1] = 1.0          # |b><b| on the low site
    cz_b = np.zeros((2, 2, 2), np.complex128)
    cz_b[0] = np.eye(2)
    cz_b[1] = np.diag([1.0, -1.0])               # Z^b on the high site
    is_a = np.zeros((4, 2, 2), np.complex128)
    is_a[0, 0, 0] = is_a[1, 1, 1] = 1.0
    is_a[2, 0, 1] = 1.0
    is_a[3, 1, 0] = 1.0
    is_b = np.zeros((4, 2, 2), np.complex128)
    is_b[0, 0, 0] = is_b[1, 1, 1] = 1.0
    is_b[2, 1, 0] = 1j
    is_b[3, 0, 1] = 1j
    return {"cz": (cz_a, cz_b), "iswap": (is_a, is_b)}


TWO_Q = _two_qubit_factors()


def edge_label(a: int, b: int) -> str:
    a, b = min(a, b), max(a, b)
    return f"e{a}_{b}"


def out_label(q: int) -> str:
    return f"out{q}"


# ---------------------------------------------------------------------------
# labelled numpy tensors + pairwise contraction (rq/tensor_core.py:338-419)


class OTensor:
    __slots__ = ("labels", "array")

    def __init__(self, labels, array):
        self.labels = tuple(labels)
        self.array = array
        assert array.ndim == len(self.labels)

    def fix(self, label, value):
        ax = self.labels.index(label)
        arr = np.take(self.array, value, axis=ax)
        if arr.ndim:
            arr = np.ascontiguousarray(arr)
        return OTensor(self.labels[:ax] + self.labels[ax + 1:], arr)

    def transpose_to(self, labels):
        labels = tuple(labels)
        if labels == self.labels:
            return self
        return OTensor(labels, permute_naive(self.array,
                                             [self.labels.index(l) for l in labels]))


def contract(a: OTensor, b: OTensor) -> OTensor:
    """Shared labels in a's order; output labels a_free + b_free."""
    bset = set(b.labels)
    shared = [l for l in a.labels if l in bset]
    for l in shared:
        if a.array.shape[a.labels.index(l)] != b.array.shape[b.labels.index(l)]:
            raise ValueError(f"dimension mismatch on {l!r}")
    out = np.tensordot(a.array, b.array,
                       axes=([a.labels.index(l) for l in shared],
                             [b.labels.index(l) for l in shared]))
    aset = set(a.labels)
    labels = [l for l in a.labels if l not in bset] + [l for l in b.labels if l not in aset]
    return OTensor(labels, np.ascontiguousarray(out) if out.ndim else np.asarray(out))


def contraction_flops(a: OTensor, b: OTensor) -> int:
    shared = set(a.labels) & set(b.labels)
    m = math.prod(d for l, d in zip(a.labels, a.array.shape) if l not in shared)
    k = math.prod(d for l, d in zip(a.labels, a.array.shape) if l in shared)
    n = math.prod(d for l, d in zip(b.labels, b.array.shape) if l not in shared)
    return 8 * m * k * n


# ---------------------------------------------------------------------------
# grid network: one tensor per site with merged edge bonds
# (rq/network_builder.py:152-289, restated as a per-site time sweep)


@dataclass
class OracleNet:
    circuit: OracleCircuit
    tensors: dict
    bond_dim: dict


def build_net(circ: OracleCircuit, in_bits: str, dtype=np.complex128) -> OracleNet:
    """All outputs open.  Per qubit: H|in>, then the cycle 1..t gates in
    time order (one bond axis per two-qubit gate, factor g[b,in,out]),
    then the final H.  Bonds of one lattice edge merge with the earliest
    activation as the most significant digit; the site's axes are its
    edges sorted by label string, then its `out` index."""
    n, t = circ.n, circ.t
    per_site = [[] for _ in range(n)]
    for cyc, name, qubits in circ.gates:
        if 0 < cyc <= t:
            for q in qubits:
                per_site[q].append((cyc, name, qubits))
    tensors = {}
    bond_count: dict = {}
    for q in range(n):
        arr = _H[:, int(in_bits[q])].copy()
        bonds = []            # (edge, bond dim) per bond axis, time order
        for cyc, name, qubits in sorted(per_site[q]):
            if len(qubits) == 1:
                arr = arr @ ONE_Q[name].T
            else:
                a, b = qubits
                fac = TWO_Q[name][0 if q == a else 1]
                arr = np.einsum("...s,bso->...bo", arr, fac)
                bonds.append(((min(a, b), max(a, b)), fac.shape[0]))
        arr = arr @ _H.T
        # group bond axes per edge, time order inside an edge
        edges = sorted({e for e, _ in bonds}, key=lambda e: edge_label(*e))
        order = []
        shape = []
        for e in edges:
            idx = [i for i, (ee, _) in enumerate(bonds) if ee == e]
            order.extend(idx)
            shape.append(math.prod(bonds[i][1] for i in idx))
            # the reference records 2^(activations) whatever the gate's
            # Schmidt rank (rq/network_builder.py:246); cut enumeration
            # follows that record, so it is mirrored here (iswap quirk)
            bond_count[e] = 1 << len(idx)
        order.append(len(bonds))      # out axis last
        shape.append(2)
        arr = np.ascontiguousarray(np.transpose(arr, order)).reshape(shape)
        labels = [edge_label(*e) for e in edges] + [out_label(q)]
        tensors[q] = OTensor(labels, arr.astype(dtype))
    return OracleNet(circ, tensors, bond_count)


def fix_outputs(net: OracleNet, bits: dict) -> OracleNet:
    tensors = dict(net.tensors)
    for q, bit in bits.items():
        tensors[q] = tensors[q].fix(out_label(q), int(bit))
    return OracleNet(net.circuit, tensors, net.bond_dim)


# ---------------------------------------------------------------------------
# plans (rq/contraction_plan.py:64-405)

_SITE = re.compile(r"t(\d+)")


@dataclass
class OraclePlan:
    lattice: str
    cuts: list           # (name, [(a,b)...], values or None)
    program: list        # ("loop", name) | ("contract", inputs, name) | ("output", name)
    batch_sites: tuple


def parse_plan(text: str) -> OraclePlan:
    lattice, cuts, program, batch = None, [], [], ()
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if tok[0] == "plan":
            lattice = tok[1]
        elif tok[0] == "batch":
            batch = tuple(int(x) for x in tok[1:])
        elif tok[0] == "cut":
            bonds, values = [], None
            for x in tok[2:]:
                if x.startswith("values="):
                    values = tuple(int(v) for v in x[7:].split(","))
                else:
                    a, b = x.split(":")
                    bonds.append(tuple(sorted((int(a), int(b)))))
            cuts.append((tok[1], bonds, values))
        elif tok[0] == "loop":
            program.append(("loop", tok[1]))
        elif tok[0] == "contract":
            arrow = tok.index("->")
            program.append(("contract", tuple(tok[1:arrow]), tok[arrow + 1]))
        elif tok[0] == "output":
            program.append(("output", tok[1]))
        else:
            raise ValueError(f"unknown statement {tok[0]!r}")
    return OraclePlan(lattice, cuts, program, batch)


def cut_dims(plan: OraclePlan, bond_dim: dict) -> tuple:
    return tuple(len(v) if v is not None else math.prod(bond_dim.get(b, 1) for b in bonds)
                 for _, bonds, v in plan.cuts)


def enumerate_paths(dims, f=1.0, seed=0, count=None):
    dims = tuple(int(d) for d in dims)
    total = math.prod(dims)
    if count is None:
        count = math.ceil(f * total)
    if count == total:
        return list(itertools.product(*(range(d) for d in dims)))
    rng = np.random.Generator(np.random.PCG64(seed))
    ids = np.sort(rng.choice(total, size=count, replace=False))
    out = []
    for pid in ids.tolist():
        p = []
        for d in reversed(dims):
            p.append(pid % d)
            pid //= d
        out.append(tuple(reversed(p)))
    return out


def _decode(cut, value, bond_dim):
    _, bonds, values = cut
    if values is not None:
        value = values[value]
    res = {}
    for b in reversed(bonds):
        d = bond_dim.get(b, 1)
        res[b] = value % d
        value //= d
    return res


class OracleExecutor:
    """Per-path plan walk with the last-value reuse cache."""

    def __init__(self, net: OracleNet, plan: OraclePlan):
        self.net, self.plan = net, plan
        site_cuts: dict = {}
        for i, (_, bonds, _) in enumerate(plan.cuts):
            for a, b in bonds:
                site_cuts.setdefault(a, []).append(i)
                site_cuts.setdefault(b, []).append(i)
        self.site_cuts = site_cuts
        defined = {}
        for st in plan.program:
            if st[0] != "contract":
                continue
            deps = set()
            for name in st[1]:
                m = _SITE.fullmatch(name)
                deps.update(site_cuts.get(int(m.group(1)), ()) if m else defined[name])
            defined[st[2]] = tuple(sorted(deps))
        self.deps = defined
        self.cut_dims = cut_dims(plan, net.bond_dim)
        self.flops = 0
        self._cache: dict = {}

    def _site(self, s, path):
        t = self.net.tensors[s]
        for i in self.site_cuts.get(s, ()):
            for bond, v in _decode(self.plan.cuts[i], path[i], self.net.bond_dim).items():
                lab = edge_label(*bond)
                if lab in t.labels:
                    t = t.fix(lab, v)
        return t

    def run(self, path) -> OTensor:
        values = {}
        for st in self.plan.program:
            if st[0] == "loop":
                continue
            if st[0] == "output":
                return values[st[1]]
            _, inputs, name = st
            key = tuple(path[i] for i in self.deps[name])
            c = self._cache.get(name)
            if c is not None and c[0] == key:
                values[name] = c[1]
                continue
            acc = None
            for inp in inputs:
                m = _SITE.fullmatch(inp)
                op = self._site(int(m.group(1)), path) if m else values[inp]
                if acc is None:
                    acc = op
                    continue
                self.flops += contraction_flops(acc, op)
                acc = contract(acc, op)
            values[name] = acc
            self._cache[name] = (key, acc)
        raise ValueError("plan has no output")


# ---------------------------------------------------------------------------
# amplitudes (rq/amplitude_engine.py:114-170)


def bits_str(value, n):
    if isinstance(value, str):
        return value
    return format(int(value), f"0{n}b")


class OracleEngine:
    def __init__(self, circuit_text: str, plan_text: str, dtype=np.complex64):
        self.circ = parse_circuit(circuit_text)
        self.plan = parse_plan(plan_text)
        self.dtype = np.dtype(dtype)
        self._nets = {}

    def base_net(self, in_bits):
        key = bits_str(in_bits, self.circ.n)
        if key not in self._nets:
            self._nets[key] = build_net(self.circ, key, self.dtype)
        return self._nets[key]

    def amplitude(self, in_bits, out_bits, f=1.0, seed=0):
        """Returns (complex amplitude, paths_total, paths_used, flops)."""
        out = bits_str(out_bits, self.circ.n)
        net = fix_outputs(self.base_net(in_bits), {q: int(b) for q, b in enumerate(out)})
        ex = OracleExecutor(net, self.plan)
        paths = enumerate_paths(ex.cut_dims, f, seed)
        total = sum(complex(ex.run(p).array[()]) for p in paths)
        return total, math.prod(ex.cut_dims), len(paths), ex.flops

    def amplitude_batch(self, in_bits, s_ab, c_sites, n_c, seed=0, f=1.0, fseed=0):
        """Returns (c_values, amplitudes ndarray, flops, paths_used)."""
        c_sites = tuple(sorted(c_sites))
        s_ab = bits_str(s_ab, self.circ.n)
        open_set = set(c_sites)
        net = fix_outputs(self.base_net(in_bits),
                          {q: int(b) for q, b in enumerate(s_ab) if q not in open_set})
        ex = OracleExecutor(net, self.plan)
        paths = enumerate_paths(ex.cut_dims, f, fseed)
        acc = None
        for p in paths:
            t = ex.run(p).transpose_to([out_label(q) for q in c_sites])
            acc = t.array.copy() if acc is None else acc + t.array
        rng = np.random.Generator(np.random.PCG64(seed))
        if n_c == 2 ** len(c_sites):
            values = np.arange(n_c)
        else:
            values = np.sort(rng.choice(2 ** len(c_sites), size=n_c, replace=False))
        return tuple(int(v) for v in values), acc.reshape(-1)[values], ex.flops, len(paths)


# ---------------------------------------------------------------------------
# dense state vector (double), for small exact checks (rq/oracle.py:51-86)


def statevector(circuit_text: str, in_bits=0) -> np.ndarray:
    circ = parse_circuit(circuit_text)
    n = circ.n
    if n > 24:
        raise ValueError("oracle state vector capped at 24 qubits")
    psi = np.zeros((2,) * n, np.complex128)
    psi[tuple(int(b) for b in bits_str(in_bits, n))] = 1.0
    cz = np.diag([1, 1, 1, -1]).astype(np.complex128).reshape(2, 2, 2, 2)
    isw = np.array([[1, 0, 0, 0], [0, 0, 1j, 0], [0, 1j, 0, 0], [0, 0, 0, 1]],
                   np.complex128).reshape(2, 2, 2, 2)
    for cyc, name, qs in circ.gates:
        if len(qs) == 1:
            psi = np.moveaxis(np.tensordot(ONE_Q[name], psi, axes=([1], [qs[0]])), 0, qs[0])
        else:
            g = cz if name == "cz" else isw
            psi = np.tensordot(g, psi, axes=([2, 3], list(qs)))
            psi = np.moveaxis(psi, [0, 1], list(qs))
    return psi.reshape(-1)
