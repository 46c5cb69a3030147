"""Build the throw-away conformance harness `conformance/` (git-ignored).

The reference's own test modules run against THIS package with `rqcsim`
aliased to it ("Conformance against the reference's own
tests").  Needs /root/reference, so it runs in the build container only; the
harness then travels to the GPU box with the gpurun snapshot, where
`scripts/conformance.sh` runs it.  Nothing here is product code and nothing
of it is committed: the reference's tests and its out-of-scope modules
(oracle / numba kernels / analysis / partition cost / CLI -- checkers and
subsystems SURVEY.md puts outside the path) are copied verbatim into the
ignored directory.
"""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
OUT = os.path.join(ROOT, "conformance")

# rqcsim modules the product replaces / reference modules kept as they are
PRODUCT = ("amplitude_engine", "circuits", "contraction_plan", "network_builder", "sampler",
           "tensor_core")
KEPT = ("oracle", "_kernels", "analysis", "partition_cost", "cli")

SHIM = '''"""rqcsim shim: the hot-path modules are paper_1811_09599_b200's."""
import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)
import paper_1811_09599_b200 as _product

for _name in %(product)r:
    _mod = importlib.import_module("paper_1811_09599_b200." + _name)
    sys.modules[__name__ + "." + _name] = _mod
    globals()[_name] = _mod
for _name in %(kept)r:
    globals()[_name] = importlib.import_module(__name__ + "." + _name)
for _name in _product.__all__:
    globals()[_name] = getattr(_product, _name)
for _mod in (analysis, partition_cost, oracle):
    for _name in dir(_mod):
        if not _name.startswith("_") and _name not in globals():
            globals()[_name] = getattr(_mod, _name)
# the reference's state-vector oracle stays the checker of its own tests
from .oracle import evolve, exact_amplitude, exact_distribution  # noqa: E402,F401
__version__ = "0.1.0"
'''


def main() -> int:
    if not os.path.isdir(REF):
        print("no /root/reference here: the harness is built in the build container", file=sys.stderr)
        return 2
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(os.path.join(OUT, "rqcsim"))
    shutil.copytree(os.path.join(REF, "tests"), os.path.join(OUT, "tests"))
    for name in KEPT:
        shutil.copy(os.path.join(REF, "src", "rqcsim", name + ".py"), os.path.join(OUT, "rqcsim"))
    with open(os.path.join(OUT, "rqcsim", "__init__.py"), "w") as fh:
        fh.write(SHIM % {"product": PRODUCT, "kept": KEPT})
    with open(os.path.join(OUT, "conftest.py"), "w") as fh:
        fh.write("import os, sys\nsys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))\n")
    print(f"wrote {OUT}: {len(os.listdir(os.path.join(OUT, 'tests')))} reference test files, "
          f"rqcsim shim over {', '.join(PRODUCT)}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
