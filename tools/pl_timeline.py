"""Plane K-pass per-tile timeline of CTA (0, 0) at S = 1024 (the largest unit, sorted first); needs a
library built with SIM_NVCC_EXTRA=-DSIM_PL_TIMELINE (sim_debug_pl_timeline)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib
from paper_2503_15078_b200 import _lib
torch.cuda.set_device(0)
sc = scenes.make_scene("cfg3")
S = 1024
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_pin_velocity(sc.pin_velocity)
s.set_contacts(sc.contacts, instance=0)
s.step(2, 5); s.synchronize()
buf = (ctypes.c_ulonglong * (4 * 64 * 8))()
_lib.lib.sim_debug_pl_timeline(buf)
a = np.array(buf, dtype=np.float64).reshape(4, 64, 8)
for p in (0, 1):
    t0 = a[p, 63, 0]; nt = int(a[p, 62, 0])
    print(f"pass {p+1}: tiles {nt}, CTA start -> (us rel.)  cols: mma[bfull, lofull0, lofull2, committed]  worker[copies, V_lo, fold, issue]")
    for t in range(min(nt, 24)):
        r = (a[p, t] - t0) / 1000.0
        print(f"  t={t:2d} " + " ".join(f"{v:7.2f}" for v in r))
