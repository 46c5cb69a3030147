"""Print the memory-stride structure of the gathered-A GEMMs of a config-2
step (which labels are rows / summed, and their element strides)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc
seen = {}
orig = tc._gather_tables
def spy(dims, labels, rows, cols, device):
    stride, acc = {}, 1
    for l, d in zip(reversed(labels), reversed(dims)):
        stride[l] = acc; acc *= d
    dim = dict(zip(labels, dims))
    key = (tuple(dims), tuple(labels), tuple(rows), tuple(cols))
    if key not in seen:
        seen[key] = 1
        print("rows", [(l, dim[l], stride[l]) for l in rows], "| k", [(l, dim[l], stride[l]) for l in cols])
    return orig(dims, labels, rows, cols, device)
tc._gather_tables = spy
lat = qf.Lattice.named("grid:5x5"); circ = qf.generate_rqc(lat, "1+24+1", 0)
eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
eng.amplitudes(0, outs)
