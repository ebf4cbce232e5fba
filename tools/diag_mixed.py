"""GPU vs oracle indicators at the GPU's own iterate, for the mixed bilateral + frictional contact
set of tests/test_gpu_contact_kinds.py: after a GPU frame of k + 1 iterations, the contact scratch
of its last iteration (theta, C diagonal; sim_debug_contact_state) was evaluated at the GPU's
(x^k, lambda^k); the oracle's indicators at the same point are compared row by row."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib
from paper_2503_15078_b200._lib import debug_contact_state
import _parity
import test_gpu_contact_kinds as T

sc, cs = T._hanging_block(1e-6, offset=float(sys.argv[1]) if len(sys.argv) > 1 else 0.001)
n = np.array([0.0, -math.sin(0.2), math.cos(0.2)])
zmin = sc.mesh.X[:, 2].min()
floor_pt = np.array([0.0, 0.0, zmin - 2e-4])
bottom = np.flatnonzero(np.abs(sc.mesh.X[:, 2] - zmin) < 1e-12)
t1, t2 = scenes.tangent_frame(n)
mixed = []
for k, v in enumerate(bottom):
    mixed.append(scenes.Contact([int(v)], [1.0], n, float(n @ floor_pt), mu=0.4, tangent1=t1, tangent2=t2))
    if k < len(cs):
        mixed.append(cs[k])
mixed += cs[len(bottom):]
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_contacts(mixed)
o = O.Oracle(sc.mesh, sc.material, sc.h)
o.set_contacts(mixed)
tol = 1e-5 * sc.mesh.bbox_diag()
x0, v0 = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
its = _parity.gpu_iterates(s, x0, v0, 5)
for k in range(1, 4):
    xk, lk = its[k - 1]
    s.set_state(x0, v0)
    s.step(1, k + 1)
    d = debug_contact_state(s)
    th_g = _parity.rows_from_triples(o, d["theta"])
    cd_g = _parity.rows_from_triples(o, d["cdiag"])
    th_o, E_o, phi_o, Jx = o.indicators(xk, x0, lk)
    kind = o.rows.kind
    cd_o = np.where(kind == 1, E_o / o.h, E_o / (o.h * o.h))
    dth = np.abs(th_g - th_o)
    dcd = np.abs(cd_g - cd_o) / np.maximum(1e-30, np.abs(cd_o))
    j = int(np.argmax(dth)); jc = int(np.argmax(dcd))
    o.lg_iters = k + 1
    xo, _, _ = o.frame(x0, v0, start=(xk, lk, k))
    o.lg_iters = 5
    print(f"iteration {k}->{k + 1}: one-step err/tol {np.abs(its[k][0] - xo).max() / tol:.4g}; max |dtheta| {dth.max():.3g} "
          f"(row {j}, kind {kind[j]}, theta_o {th_o[j]:.6g}, lam {lk[j]:.4g}); max rel dC {dcd.max():.3g} (row {jc}, "
          f"kind {kind[jc]}, C_o {cd_o[jc]:.6g}, C_g {cd_g[jc]:.6g}, lam {lk[jc]:.4g})", flush=True)
