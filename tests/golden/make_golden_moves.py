"""Golden L/R move lists of the reference's plan_permutation
(rq/tensor_core.py:81-206), written by importing the reference in the build
container:  python tests/golden/make_golden_moves.py  ->  golden_moves.json"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from rqcsim import tensor_core as rq  # noqa: E402


def main():
    rng = np.random.Generator(np.random.PCG64(1811))
    cases = [([2] * 7, [2, 5, 4, 0, 3, 6, 1], 2, 4),
             ([2] * 10, [1, 0, 2, 3, 4, 5, 6, 7, 8, 9], 5, 8),
             ([2] * 10, [0, 1, 2, 3, 4, 5, 6, 7, 9, 8], 5, 8),
             ([2, 2, 2], [0, 1, 2], 5, 10)]
    while len(cases) < 400:
        k = int(rng.integers(1, 13))
        dims = [int(rng.integers(1, 7)) for _ in range(k)]
        perm = [int(v) for v in rng.permutation(k)]
        mu = int(rng.integers(0, 8))
        cases.append((dims, perm, mu, mu + int(rng.integers(0, 8))))
    out = []
    for dims, perm, mu, nu in cases:
        plan = rq.plan_permutation(dims, perm, mu, nu)
        out.append({"dims": dims, "perm": perm, "mu": mu, "nu": nu, "fallback": plan.fallback,
                    "moves": [[m.kind, list(m.group_perm), m.gamma] for m in plan.moves]})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_moves.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {len(out)} cases to {path}")


if __name__ == "__main__":
    main()
