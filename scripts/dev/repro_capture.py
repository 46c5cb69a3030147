"""Find the call that invalidates the single-call graph capture (debug)."""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import _lib

from cuda.bindings import runtime as rt
orig = _lib.check
state = {"bad": False}

def status():
    s = torch.cuda.current_stream().cuda_stream
    err, st = rt.cudaStreamIsCapturing(s)
    return (int(err), int(st))

def check(st, what):
    if not state["bad"]:
        r = status()
        if r[1] == 2 or r[0] != 0:
            state["bad"] = True
            print("FIRST INVALIDATED after/before library call:", what, r, flush=True)
            traceback.print_stack(limit=14)
    return orig(st, what)

import paper_1811_09599_b200.tensor_core as tcore
_lib.check = check

class Proxy:
    def __init__(self, lib): self._lib = lib
    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if not name.startswith("qf_"): return fn
        def w(*a):
            pre = status() if not state["bad"] else None
            r = fn(*a)
            if not state["bad"]:
                post = status()
                if post[1] == 2 or post[0] != 0:
                    state["bad"] = True
                    print("INVALIDATED", "inside" if pre and pre[1] == 1 else "before", name, pre, post, "rc", r, [x if isinstance(x,(int,float)) else "*" for x in a], flush=True)
            return r
        return w
real = _lib.load()
prox = Proxy(real)
_lib.load = lambda path=None: prox
odb = tcore.device_buffer
def db(*a, **k):
    pre = status() if not state["bad"] else None
    r = odb(*a, **k)
    if not state["bad"]:
        post = status()
        if post[1] == 2 or post[0] != 0:
            state["bad"] = True
            print("INVALIDATED in device_buffer", pre, post, a, flush=True)
    return r
tcore.device_buffer = db
import paper_1811_09599_b200.tensor_core as tcore
for mod in (tcore,):
    pass
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
            state["bad"] = False
            try:
                vals = [eng.amplitude(0, int(o))[0] for o in outs]
                print("ok  ", kind, depth, np.dtype(dt).name, flush=True)
            except Exception as e:
                print("FAIL", kind, depth, np.dtype(dt).name, repr(e)[:300], flush=True)
                torch.cuda.synchronize()
