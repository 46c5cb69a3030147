"""Which criterion-1 style single amplitude() calls fail under graph replay."""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1811_09599_b200 as qf

grids = ["grid:1x2", "grid:2x2", "grid:4x4", "grid:4x5", "bristlecone-24"]
depths = ["1+8+1", "1+16+1", "1+24+1"]
rng = np.random.default_rng(2024)
for kind in grids:
    for depth in depths:
        for dt in (np.complex64, np.complex128):
            lat = qf.Lattice.named(kind)
            circ = qf.generate_rqc(lat, depth, seed=0)
            eng = qf.AmplitudeEngine(circ, dtype=dt)
            outs = rng.integers(0, 2 ** circ.n, size=3)
            try:
                vals = [eng.amplitude(0, int(o))[0] for o in outs]
                print("ok  ", kind, depth, np.dtype(dt).name, flush=True)
            except Exception as e:
                print("FAIL", kind, depth, np.dtype(dt).name, repr(e)[:300], flush=True)
                traceback.print_exc(limit=12)
                torch.cuda.synchronize()
