"""Run a few cfg3 frames (no bench extras) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 3
name = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
torch.cuda.set_device(0)
sc = scenes.make_scene(name)
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_pin_velocity(sc.pin_velocity)
packed = s.pack_contacts(sc.contacts)
for f in range(frames):
    s.set_contacts(packed=packed)
    s.step(1, 5)
s.synchronize()
print("done", s.stats()["kernels_per_frame"])
x, v = s.get_state()
print("max|x-X|", float(np.abs(x - sc.mesh.X).max()), "finite", bool(np.isfinite(x).all()), "max|v|", float(np.abs(v).max()))
from paper_2503_15078_b200._lib import debug_cr_timeline
tl = debug_cr_timeline(s)
print("CR timeline us:", " ".join(f"{v:.1f}" for v in tl[:12]), "| it3: start %.1f W %.1f mv %.1f wait %.1f Sv %.1f end %.1f" % tuple(tl[12:18]), "| end", f"{tl[20]:.1f} {tl[21]:.1f}", "na", int(tl[31]), "sub", " ".join(f"{v:.1f}" for v in tl[22:29]))
from paper_2503_15078_b200._lib import lib as _L
