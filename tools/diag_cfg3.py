"""Diagnose GPU-vs-oracle differences on cfg3 (run on the GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib

torch.cuda.set_device(0)
sc = scenes.make_scene("cfg3")
tol = 1e-5 * sc.mesh.bbox_diag()
x0, v0 = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
pins = x0[sc.mesh.fixed.astype(bool)] + sc.h * sc.pin_velocity
print("tol", tol, flush=True)

def gpu_frame(contacts, iters):
    s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    s.set_pin_velocity(sc.pin_velocity)
    if contacts:
        s.set_contacts(contacts)
    s.step(1, iters)
    x, v = s.get_state()
    lam = s.get_lambda() if contacts else None
    G = s.debug_delassus() if contacts else None
    s.close()
    return x, lam, G

# (a) no contacts
o = O.Oracle(sc.mesh, sc.material, sc.h)
xo, _, _ = o.frame(x0, v0, pin_targets=pins)
xg, _, _ = gpu_frame([], 5)
print("(a) no contacts 5 it: max dx", np.abs(xg - xo).max(), flush=True)
# (b) contacts
o.set_contacts(sc.contacts)
cv, G = None, None
for iters in (1, 2, 5):
    o.lg_iters = iters
    xo, _, info = o.frame(x0, v0, pin_targets=pins)
    xg, lg, (cv, G) = gpu_frame(sc.contacts, iters)
    d = np.abs(xg - xo)
    print(f"(b) contacts {iters} it: max dx {d.max():.3e} argmax vertex {np.unravel_index(d.argmax(), d.shape)}; "
          f"lam max diff {np.abs(lg - info['lam']).max():.3e} of {np.abs(info['lam']).max():.3e}", flush=True)
order = {int(v): i for i, v in enumerate(o.vc)}
idx = np.array([order[int(v)] for v in cv])
Go = o.G[np.ix_(idx, idx)]
print("(c) G rel err", np.abs(G - Go).max() / np.abs(Go).max(), "diag rel err", np.abs(np.diag(G) - np.diag(Go)).max() / np.abs(np.diag(Go)).max(), flush=True)
bad = np.argwhere(np.abs(G - Go) > 1e-4 * np.abs(Go).max())
print("   bad entries", len(bad), bad[:10], flush=True)
