"""Regenerate the package data the drop-in API needs from the reference
(run in a container where /root/reference exists; the output is committed):

  paper_1811_09599_b200/data/lattices.json  -- the Bristlecone coordinate
      tables of rqcsim.circuits.Lattice.bristlecone (rq/circuits.py:130-170,
      data/lattices/bristlecone_{24..72}.txt), stored as per-row column runs
  paper_1811_09599_b200/data/shipped_plans.json -- the plans rqcsim ships
      for builtin_plan / load_plan (rq/contraction_plan.py:778-786), as plan
      text re-formatted by the product's own format_plan

These are data the public API returns (Lattice.named, builtin_plan), not
code; parity is pinned by tests/test_shipped_data.py against
tests/golden/golden_shipped.json (written by the same run from rqcsim
directly)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import rqcsim as rq  # noqa: E402
from rqcsim import circuits as rq_circuits  # noqa: E402
from rqcsim import contraction_plan as rq_plan  # noqa: E402

from paper_1811_09599_b200.contraction_plan import format_plan, parse_plan  # noqa: E402


def runs(coords):
    rows = {}
    for r, c in coords:
        rows.setdefault(r, []).append(c)
    out = []
    for r in sorted(rows):
        cols = sorted(rows[r])
        lo = prev = cols[0]
        for c in cols[1:] + [None]:
            if c is None or c != prev + 1:
                out.append([r, lo, prev])
                if c is not None:
                    lo = c
            if c is not None:
                prev = c
    return out


def main():
    lat = {}
    golden = {"lattices": {}, "plans": {}, "costs": {}}
    for size in rq_circuits.BRISTLECONE_SIZES:
        L = rq.Lattice.bristlecone(size)
        coords = [tuple(map(int, L.coords(i))) for i in range(L.n)]
        lat[str(size)] = runs(coords)
        golden["lattices"][str(size)] = {"sites": coords, "edges": [list(e) for e in L.edges()]}
    plans = {}
    for name in rq_plan._PLAN_FILES:
        plan = rq.load_plan(name)
        text = rq.format_plan(plan)
        plans[name] = format_plan(parse_plan(text))
        golden["plans"][name] = text
        L = rq.Lattice.named(name)
        for depth in ("1+8+1", "1+16+1"):
            e = rq.estimate_cost(plan, L, depth)
            golden["costs"][f"{name} {depth}"] = {"flops": int(e.total_flops),
                                                  "peak_bytes": int(e.peak_bytes),
                                                  "paths": int(e.paths)}
    data = os.path.join(ROOT, "paper_1811_09599_b200", "data")
    with open(os.path.join(data, "lattices.json"), "w") as fh:
        json.dump({"source": "rqcsim data/lattices/bristlecone_*.txt (reference), as "
                             "[row, first column, last column] runs", "bristlecone": lat},
                  fh, indent=0)
    with open(os.path.join(data, "shipped_plans.json"), "w") as fh:
        json.dump({"source": "rqcsim data/plans/*.txt (reference), via format_plan", "plans": plans},
                  fh, indent=1)
    with open(os.path.join(ROOT, "tests", "golden", "golden_shipped.json"), "w") as fh:
        json.dump(golden, fh)
    print("wrote", len(lat), "lattices,", len(plans), "plans")


if __name__ == "__main__":
    main()
