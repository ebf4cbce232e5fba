"""Conditioning of the method's frame map, measured on the fp64 oracle alone: for each frame of a
scene (or a cfg5 instance), the oracle's frame from (x_t, v_t) and from the same state rounded to
fp32; the per-iteration max |x^k - x^k_rounded| / (1e-5 bbox diagonal).  A frame whose value at the
last iteration approaches 1 cannot be reproduced to the north-star tolerance by any fp32
computation: rounding alone moves the exact result by that much.
usage: python tools/frame_conditioning.py [cfg3 | <cfg5 instance>] [frames] [--cr N] [--mu0]"""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import scenes
from oracle import oracle as O

args = [a for a in sys.argv[1:] if not a.startswith("--")]
which = args[0] if args else "cfg3"
frames = int(args[1]) if len(args) > 1 else 3
cr = int(sys.argv[sys.argv.index("--cr") + 1]) if "--cr" in sys.argv else 10
sc = scenes.make_scene("cfg3")
tol = 1e-5 * sc.mesh.bbox_diag()
if which == "cfg3":
    cs, v = sc.contacts, np.zeros_like(sc.mesh.X)
else:
    v, cs = scenes.batch_instance(sc, int(which))
if "--mu0" in sys.argv:
    cs = [dataclasses.replace(c, mu=0.0) for c in cs]
o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=5, cr_iters=cr)
o.set_contacts(cs)
x = sc.mesh.X.copy()
r32 = lambda a: a.astype(np.float32).astype(np.float64)
for f in range(frames):
    xa, va, ia = o.frame(x, v, pin_targets=x[o.pinned] + sc.h * sc.pin_velocity, capture=True)
    xr, vr = r32(x), r32(v)
    xb, _, ib = o.frame(xr, vr, pin_targets=xr[o.pinned] + sc.h * sc.pin_velocity, capture=True)
    e = [float(np.abs(a["x_next"] - b["x_next"]).max() / tol) for a, b in zip(ia["iters"], ib["iters"])]
    print(f"{which} frame {f}: fp32-input sensitivity per iteration (x / 1e-5 bbox): "
          + " ".join(f"{q:.4f}" for q in e), flush=True)
    x, v = xa, va
