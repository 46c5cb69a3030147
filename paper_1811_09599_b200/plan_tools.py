"""Plan tooling: cost a plan for any path subset,
reorder region contractions greedily by flops, and choose sliced bonds
(waist or internal) so that a plan fits a memory budget.

All of it is host-side shape arithmetic on the plan language of
`contraction_plan` (rq/contraction_plan.py:12-17); nothing here touches the
device.  The costs follow the reference's conventions: 8*m*k*n flops per
pairwise contraction, inputs folded left to right
(rq/contraction_plan.py:509-516), a step re-executed whenever the values of
its cut dependencies differ from the previous path's (last-value reuse,
rq/contraction_plan.py:477-523), sliced bonds of dimension 1 in the site
tensors (rq/contraction_plan.py:566-644).
"""

from __future__ import annotations

import math
from typing import Iterable, Optional, Sequence

from .circuits import DepthSpec, Lattice, edge_activations
from .contraction_plan import (ContractionPlan, ContractStep, PlanError, _SITE_RE, enumerate_paths,
                               estimate_cost, two_region_plan)
from .network_builder import edge_label, out_label


def bond_dims(lattice: Lattice, depth) -> dict:
    """Bond dimension 2^(activations) of every active lattice edge."""
    t = DepthSpec.parse(depth).t
    return {e: 2 ** k for e, k in edge_activations(lattice, t).items() if k > 0}


def path_subset_flops(plan: ContractionPlan, lattice: Lattice, depth, paths: Iterable,
                      *, open_sites: Sequence[int] = ()) -> int:
    """Flops of walking `paths` in the given order under last-value reuse --
    what PathStats.flops reports for an amplitude computed from exactly that
    path list (f < 1 subsets, one rank's shard, ...).  For the full
    lexicographic list it equals estimate_cost(...).total_flops."""
    est = estimate_cost(plan, lattice, depth, open_sites=open_sites)
    analysis = plan.analyze(lattice)
    step_flops = {s.name: s.flops for s in est.steps}
    last: dict = {}
    total = 0
    for path in paths:
        path = tuple(path)
        for step in plan.steps():
            key = tuple(path[i] for i in analysis.step_deps[step.name])
            if last.get(step.name) != key:
                last[step.name] = key
                total += step_flops[step.name]
    return total


def fidelity_flops(plan: ContractionPlan, lattice: Lattice, depth, f: float = 1.0, seed: int = 0,
                   *, open_sites: Sequence[int] = ()) -> int:
    """Flops of one amplitude at fidelity f (the seeded path draw of
    FidelitySpec / enumerate_paths)."""
    dims = plan.cut_dims(bond_dims(lattice, depth))
    return path_subset_flops(plan, lattice, depth, enumerate_paths(dims, f=f, seed=seed),
                             open_sites=open_sites)


# ---------------------------------------------------------------------------
# greedy contraction order


def _site_shape(lattice: Lattice, site: int, bonds: dict, sliced: set, opened: set) -> dict:
    shape = {edge_label(*e): d for e, d in bonds.items() if site in e}
    for l in shape.keys() & sliced:
        shape[l] = 1
    if site in opened:
        shape[out_label(site)] = 2
    return shape


def _fold_cost(acc: dict, op: dict) -> tuple:
    common = acc.keys() & op.keys()
    m = math.prod(d for l, d in acc.items() if l not in common)
    k = math.prod(d for l, d in acc.items() if l in common)
    n = math.prod(d for l, d in op.items() if l not in common)
    out = {l: d for l, d in acc.items() if l not in common}
    out.update((l, d) for l, d in op.items() if l not in common)
    return 8 * m * k * n, out


def greedy_order(lattice: Lattice, sites: Sequence[int], bonds: dict, *, start=None,
                 sliced: Iterable[str] = (), open_sites: Sequence[int] = ()) -> tuple:
    """Left-to-right fold order for a set of sites: from `start` (a shape
    dict of an intermediate, or None to try every site first) absorb, at
    each step, the site whose contraction costs the fewest flops (ties: the
    smaller result, then the lower id).  Returns (order, flops)."""
    sliced, opened = set(sliced), set(open_sites)
    shapes = {s: _site_shape(lattice, s, bonds, sliced, opened) for s in sites}
    best = None
    firsts = [None] if start is not None else sorted(sites)
    for first in firsts:
        acc = dict(start) if start is not None else dict(shapes[first])
        todo = set(sites) - ({first} if first is not None else set())
        order = [first] if first is not None else []
        flops = 0
        while todo:
            cands = []
            for s in todo:
                f, out = _fold_cost(acc, shapes[s])
                touching = bool(acc.keys() & shapes[s].keys())
                cands.append((not touching, f, math.prod(out.values()), s, out))
            _, f, _, s, out = min(cands, key=lambda c: c[:4])
            flops += f
            acc = out
            order.append(s)
            todo.discard(s)
        if best is None or flops < best[1]:
            best = (tuple(order), flops)
    return best


def reorder_plan(plan: ContractionPlan, lattice: Lattice, depth,
                 *, open_sites: Sequence[int] = ()) -> ContractionPlan:
    """The same plan (regions, cuts, loops, step names, reuse) with each
    step's site inputs re-ordered greedily by flops.  A step that starts
    from an intermediate keeps it first; a step is only changed when the
    greedy order is strictly cheaper than the given one."""
    bonds = bond_dims(lattice, depth)
    sliced = {edge_label(*b) for c in plan.cuts for b in c.bonds}
    est = estimate_cost(plan, lattice, depth, open_sites=open_sites)
    shapes: dict = {}
    old_flops = {s.name: s.flops for s in est.steps}
    opened = set(open_sites)
    program = []
    for kind, payload in plan.program:
        if kind != "contract":
            program.append((kind, payload))
            continue
        step = payload
        sites = [int(x[1:]) for x in step.inputs if _SITE_RE.fullmatch(x)]
        inter = [x for x in step.inputs if not _SITE_RE.fullmatch(x)]
        new = step
        if len(sites) >= 2 and len(inter) <= 1 and (not inter or step.inputs[0] == inter[0]):
            start = None
            if inter:
                start = shapes[inter[0]]
            order, flops = greedy_order(lattice, sites, bonds, start=start, sliced=sliced,
                                        open_sites=open_sites)
            if flops < old_flops[step.name]:
                new = ContractStep(tuple(inter) + tuple(f"t{s}" for s in order), step.name,
                                   step.reuse)
        # shape of the step's result (independent of the fold order)
        acc = None
        for x in new.inputs:
            m = _SITE_RE.fullmatch(x)
            op = _site_shape(lattice, int(m.group(1)), bonds, sliced, opened) if m else shapes[x]
            acc = dict(op) if acc is None else _fold_cost(acc, op)[1]
        shapes[step.name] = acc
        program.append(("contract", new))
    return ContractionPlan(plan.lattice_kind, plan.cuts, tuple(program), plan.batch_sites)


# ---------------------------------------------------------------------------
# slicing for a memory budget


def slice_for_budget(lattice: Lattice, depth, region_a, region_b, region_c, budget_bytes: int,
                     *, candidates: Optional[Sequence] = None, itemsize: int = 8,
                     max_cuts: int = 8, reorder: bool = True) -> ContractionPlan:
    """A two-region plan (two_region_plan) whose peak live set
    (estimate_cost) fits `budget_bytes`: bonds are cut one at a time -- the
    A|B waist or bonds inside a region ("internal sub-slicing"; their sum
    is the path sum) -- each time the candidate that lowers the peak most
    (ties: fewer total flops).  Raises PlanError if `max_cuts` cuts do not
    reach the budget."""
    bonds = bond_dims(lattice, depth)
    if candidates is None:
        candidates = sorted(bonds)
    cands = [tuple(sorted(b)) for b in candidates if tuple(sorted(b)) in bonds]
    cuts: list = []

    def build(cs):
        p = two_region_plan(lattice, region_a, region_b, region_c, cs)
        if reorder:
            p = reorder_plan(p, lattice, depth)
        return p, estimate_cost(p, lattice, depth, itemsize=itemsize)

    plan, est = build(cuts)
    while est.peak_bytes > budget_bytes:
        if len(cuts) >= max_cuts:
            raise PlanError(f"peak {est.peak_bytes} B still above budget {budget_bytes} B "
                            f"after {len(cuts)} cuts")
        best = None
        for b in cands:
            if b in cuts:
                continue
            try:
                p, e = build(cuts + [b])
            except PlanError:
                continue
            score = (e.peak_bytes, e.total_flops, b)
            if best is None or score < best[0]:
                best = (score, b, p, e)
        if best is None:
            raise PlanError("no bond left to cut")
        _, b, plan, est = best
        cuts.append(b)
    return plan
