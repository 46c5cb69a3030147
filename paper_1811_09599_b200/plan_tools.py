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


# ---------------------------------------------------------------------------
# exact contraction trees (subset dynamic programming)
#
# The reference orders a region greedily (rq/contraction_plan.py:651-673:
# grow a cluster from the lowest site id, always absorbing the neighbour
# that keeps the open-bond count smallest) and contracts it left to right.
# At full depth that order is infeasible for the big regions (2^35..2^50
# entries).  `tree_order` finds the contraction TREE with the
# fewest flops among all trees of connected sub-regions whose intermediates
# stay <= 2^cap entries, by dynamic programming over subsets of the region
# (bitmasks; log2 sizes are integers since every bond is a power of two):
#     best[S] = min over S = S1 + S2 (both connected, S1 holds S's lowest
#               member) of best[S1] + best[S2] + 8 * 2^((lg S1 + lg S2 + lg S) / 2)
# where lg X is log2 of the entries of X's open bonds -- the labels of the
# pairwise contraction are the union of both operands' labels, whose log
# size is (lg S1 + lg S2 + lg S) / 2.  Regions above EXACT_MAX members are
# split in two halves along the lattice's longer axis, each half solved
# by a beam search over sequential (left-deep) orders under the same cap:
# states are connected sub-regions (deduplicated, cheapest prefix kept),
# each extended by every neighbouring site whose result fits, the `beam`
# cheapest kept per length.

EXACT_MAX = 18


def _lg(d: int) -> int:
    v = int(d).bit_length() - 1
    if d < 1 or (1 << v) != d:
        raise PlanError(f"bond dimension {d} is not a power of two")
    return v


def _items_tables(items: Sequence[dict]):
    """Per-label item masks and log sizes; item adjacency (shared labels)."""
    import numpy as np
    n = len(items)
    where: dict = {}
    for i, it in enumerate(items):
        for l, d in it.items():
            w = where.setdefault(l, [0, _lg(d)])
            w[0] |= 1 << i
    adj = [0] * n
    for l, (m, _) in where.items():
        members = [i for i in range(n) if (m >> i) & 1]
        if len(members) > 2:
            raise PlanError(f"label {l!r} joins {len(members)} tensors (hyper-edge)")
        if len(members) == 2:
            a, b = members
            adj[a] |= 1 << b
            adj[b] |= 1 << a
    masks = np.arange(1 << n, dtype=np.int64)
    lg = np.zeros(1 << n, dtype=np.int64)
    for l, (m, w) in where.items():
        if w == 0:
            continue
        bits = [i for i in range(n) if (m >> i) & 1]
        cnt = sum((masks >> b) & 1 for b in bits)
        lg += np.where(cnt == 1, w, 0)
    # connectivity: flood from the lowest member inside the mask
    low = masks & -masks
    reach = low.copy()
    for _ in range(n):
        grown = reach.copy()
        for i in range(n):
            grown |= np.where((reach >> i) & 1, adj[i], 0)
        grown &= masks
        if np.array_equal(grown, reach):
            break
        reach = grown
    connected = reach == masks
    return lg, connected


def _dp_tree(items: Sequence[dict], cap: Optional[int]):
    """(flops, tree) of the cheapest connected-split tree over `items`
    whose proper intermediates have log2 size <= cap (None: no cap); tree
    leaves are item indices."""
    import numpy as np
    n = len(items)
    if n == 1:
        return 0, 0
    lg, connected = _items_tables(items)
    full = (1 << n) - 1
    ok = connected.copy()
    if cap is not None:
        ok &= lg <= cap
        ok[full] = connected[full]
    best = np.full(1 << n, np.inf)
    split = np.zeros(1 << n, dtype=np.int64)
    for i in range(n):
        best[1 << i] = 0.0
    # combos[k]: every k-bit pattern as rows of 0/1, for depositing onto a mask
    combos = {}
    cand = np.nonzero(ok)[0]
    cand = cand[(cand & (cand - 1)) != 0]            # at least two members
    for mask in cand.tolist():
        pos = [i for i in range(n) if (mask >> i) & 1]
        k = len(pos)
        c = combos.get(k)
        if c is None:
            r = np.arange(1, 1 << k, 2, dtype=np.int64)   # patterns holding the lowest member
            r = r[r != (1 << k) - 1]
            c = combos[k] = ((r[:, None] >> np.arange(k)) & 1)
        sub = c @ (np.int64(1) << np.array(pos, dtype=np.int64))
        rest = mask ^ sub
        val = best[sub] + best[rest]
        good = ok[sub] & ok[rest] & np.isfinite(val)
        if not good.any():
            continue
        cost = 8.0 * np.exp2((lg[sub] + lg[rest] + lg[mask]) // 2)
        tot = np.where(good, val + cost, np.inf)
        j = int(np.argmin(tot))
        if tot[j] < best[mask]:
            best[mask] = tot[j]
            split[mask] = sub[j]
    if not np.isfinite(best[full]):
        raise PlanError(f"no contraction tree keeps every intermediate <= 2^{cap} entries")

    def tree(m):
        if m & (m - 1) == 0:
            return m.bit_length() - 1
        s = int(split[m])
        return (tree(s), tree(m ^ s))

    return int(best[full]), tree(full)


def tree_order(lattice: Lattice, sites: Sequence[int], bonds: dict, *, sliced: Iterable[str] = (),
               open_sites: Sequence[int] = (), cap_log2: Optional[int] = 30,
               beam: int = 2048) -> tuple:
    """The cheapest contraction tree of a region (see the section comment):
    returns (flops, tree) with leaves = site ids.  Bonds in `sliced` have
    dimension 1 (a path fixes their value); open sites carry their `out`
    index.  Regions above EXACT_MAX sites: beam search over left-deep
    (sequential) trees instead (_beam_chain)."""
    sliced, opened = set(sliced), set(open_sites)
    sites = list(sites)
    shapes = [_site_shape(lattice, s, bonds, sliced, opened) for s in sites]
    if len(sites) <= EXACT_MAX:
        flops, t = _dp_tree(shapes, cap_log2)
    else:
        flops, t = _beam_chain(shapes, cap_log2, beam)
    def relabel(t):
        return sites[t] if isinstance(t, int) else (relabel(t[0]), relabel(t[1]))

    return flops, relabel(t)


def _beam_chain(items: Sequence[dict], cap: Optional[int], beam: int):
    """(flops, left-deep tree) of the best sequential order found by a beam
    search over connected prefixes whose results stay <= 2^cap entries."""
    n = len(items)
    lab_items: dict = {}
    for i, it in enumerate(items):
        for l in it:
            lab_items.setdefault(l, []).append(i)
    nbr = [set() for _ in range(n)]
    for l, ii in lab_items.items():
        if len(ii) == 2:
            nbr[ii[0]].add(ii[1])
            nbr[ii[1]].add(ii[0])
    lgd = [{l: _lg(d) for l, d in it.items()} for it in items]

    def open_labels(mask_members):
        out = {}
        for i in mask_members:
            for l, w in lgd[i].items():
                if l in out:
                    del out[l]
                else:
                    out[l] = w
        return out

    states = {}
    for i in range(n):
        states[1 << i] = (0, (i,), dict(lgd[i]))
    for _ in range(n - 1):
        nxt = {}
        for mask, (fl, order, acc) in states.items():
            frontier = set().union(*(nbr[i] for i in order)) - set(order)
            for j in frontier:
                common = acc.keys() & lgd[j].keys()
                lg_mkn = sum(acc.values()) + sum(w for l, w in lgd[j].items() if l not in common)
                out = {l: w for l, w in acc.items() if l not in common}
                out.update((l, w) for l, w in lgd[j].items() if l not in common)
                nm = mask | (1 << j)
                if cap is not None and nm != (1 << n) - 1 and sum(out.values()) > cap:
                    continue
                cand = (fl + 8 * 2 ** lg_mkn, order + (j,), out)
                if nm not in nxt or cand[0] < nxt[nm][0]:
                    nxt[nm] = cand
        if not nxt:
            raise PlanError(f"no sequential order keeps every intermediate <= 2^{cap} entries")
        states = dict(sorted(nxt.items(), key=lambda kv: kv[1][0])[:beam])
    fl, order, _ = min(states.values(), key=lambda v: v[0])
    t = order[0]
    for j in order[1:]:
        t = (t, j)
    return int(fl), t


def _tree_sites(t) -> list:
    return [t] if isinstance(t, int) else _tree_sites(t[0]) + _tree_sites(t[1])


def _chain(t, emit) -> list:
    """Fold inputs for tree t: a site extends the chain of its sibling; of
    two composite children the smaller becomes its own named step."""
    if isinstance(t, int):
        return [f"t{t}"]
    a, b = t
    if isinstance(b, int):
        return _chain(a, emit) + [f"t{b}"]
    if isinstance(a, int):
        return _chain(b, emit) + [f"t{a}"]
    if len(_tree_sites(a)) < len(_tree_sites(b)):
        a, b = b, a
    return _chain(a, emit) + [emit(b)]


def tree_plan(plan: ContractionPlan, lattice: Lattice, depth, *, open_sites: Sequence[int] = (),
              cap_log2: Optional[int] = 30) -> ContractionPlan:
    """A slice-first plan with the same cuts, batch region and joins as
    `plan` (e.g. a shipped plan): every region -- the sites one chain of
    steps folds in, from its first step through the steps that extend it --
    is contracted as the cheapest tree of tree_order with its cut bonds
    sliced, each sub-step placed right after the loop of the last cut it
    depends on (hoisted out of the inner loops otherwise, reuse
    global/outer), and the joins (steps combining two or more region
    values) kept as they are."""
    bonds = bond_dims(lattice, depth)
    sliced = {edge_label(*b) for c in plan.cuts for b in c.bonds}
    cut_of = {}
    for i, c in enumerate(plan.cuts):
        for b in c.bonds:
            for s in b:
                cut_of.setdefault(s, set()).add(i)
    steps = list(plan.steps())
    inter = {s.name for s in steps}
    # region chains: a step with at most one intermediate input extends it
    region_of: dict = {}
    regions: dict = {}
    joins = []
    for st in steps:
        ins_i = [x for x in st.inputs if x in inter]
        sites = [int(x[1:]) for x in st.inputs if _SITE_RE.fullmatch(x)]
        if len(ins_i) >= 2 or (len(ins_i) == 1 and ins_i[0] not in region_of):
            joins.append(st)
            continue
        root = region_of[ins_i[0]] if ins_i else st.name
        regions.setdefault(root, []).extend(sites)
        region_of[st.name] = root
    final = {}
    for st in steps:
        if st.name in region_of:
            final[region_of[st.name]] = st.name      # the chain's last name wins
    program_by_level: dict = {}
    names = set()

    def deps_of_sites(ss):
        d = set()
        for s in ss:
            d |= cut_of.get(s, set())
        return d

    def place(inputs, name, deps):
        level = (max(deps) + 1) if deps else 0
        reuse = "global" if not deps else ("outer" if len(deps) < len(plan.cuts) else None)
        program_by_level.setdefault(level, []).append(ContractStep(tuple(inputs), name, reuse))

    for root, sites in regions.items():
        _, t = tree_order(lattice, sites, bonds, sliced=sliced, open_sites=open_sites,
                          cap_log2=cap_log2)
        out_name = final[root]
        counter = [0]

        def emit(sub, out_name=out_name, counter=counter):
            ins = _chain(sub, emit)
            counter[0] += 1
            nm = f"{out_name}_{counter[0]}"
            while nm in inter or nm in names:
                counter[0] += 1
                nm = f"{out_name}_{counter[0]}"
            names.add(nm)
            place(ins, nm, deps_of_sites(_tree_sites(sub)))
            return nm

        ins = _chain(t, emit)
        place(ins, out_name, deps_of_sites(sites))
    region_deps = {final[r]: deps_of_sites(s) for r, s in regions.items()}
    for st in joins:
        d = set()
        for x in st.inputs:
            m = _SITE_RE.fullmatch(x)
            d |= cut_of.get(int(m.group(1)), set()) if m else region_deps.get(x, set())
        region_deps[st.name] = d
        place(st.inputs, st.name, d)
    program = list(program_by_level.get(0, []))
    program = [("contract", s) for s in program]
    for i, c in enumerate(plan.cuts):
        program.append(("loop", c.name))
        program.extend(("contract", s) for s in program_by_level.get(i + 1, []))
    program.append(("output", plan.analyze(lattice).output_name))
    out = ContractionPlan(plan.lattice_kind, plan.cuts, tuple(program), plan.batch_sites)
    out.analyze(lattice)
    return out
