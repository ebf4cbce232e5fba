"""Conditioning of the incline-block frame with random per-vertex initial velocities: the oracle's own
sensitivity to fp32 input rounding vs the GPU error at S = 1 / 3 / 96."""
import math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenes, paper_2503_15078_b200 as sl
from oracle import oracle as O
from _parity import sensitivity
sc = scenes.incline_block(theta_deg=10.0, mu=math.tan(math.radians(10.0)) - 0.05, nv=5, edge=0.1, youngs=1e8)
v0 = scenes.random_state(sc.mesh, seed=0, amp=0.02)[1]
tol = 1e-5 * sc.mesh.bbox_diag()
o = O.Oracle(sc.mesh, sc.material, sc.h); o.set_contacts(sc.contacts)
xo, _, _ = o.frame(sc.mesh.X.copy(), v0)
print("sens/tol", sensitivity(o, sc.mesh.X, v0, xo) / tol)
for S in (1, 3, 96):
    s = sl.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
    s.set_contacts_batch([sc.contacts] * S)
    s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), np.broadcast_to(v0, (S,) + v0.shape))
    s.step(1, 5)
    P = s.get_positions()
    print("S", S, "err/tol", np.abs(P[0] - xo).max() / tol)
