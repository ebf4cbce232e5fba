"""Per-iteration divergence of one scene, GPU (n_instances = 1) vs the fp64 oracle: for
k = 1..iters, one frame of k L-G iterations from the same (x, v, lambda = 0) on both sides;
prints max |x_gpu - x_oracle| / (1e-5 bbox) and, at the last iteration, the rows whose
theta differ.  usage: python tools/diag_instance.py cfg5 <instance> [iters]
                      python tools/diag_instance.py incline [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib
from paper_2503_15078_b200._lib import debug_contact_state
import _parity

what = sys.argv[1]
if what == "cfg5":
    sc = scenes.make_scene("cfg3")
    inst = int(sys.argv[2])
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    v0, cs = scenes.batch_instance(sc, inst)
    x0 = sc.mesh.X.copy()
else:
    import math
    sc = scenes.incline_block(theta_deg=10.0, mu=math.tan(math.radians(10.0)) + 0.05, nv=5, edge=0.1, youngs=1e8)
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    v0, cs = np.zeros_like(sc.mesh.X), sc.contacts
    x0 = sc.mesh.X.copy()
tol = 1e-5 * sc.mesh.bbox_diag()
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_pin_velocity(sc.pin_velocity)
s.set_contacts(cs)
for k in range(1, iters + 1):
    s.set_state(x0, v0)
    s.step(1, k)
    xg, _ = s.get_state()
    st = debug_contact_state(s)
    o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=k)
    o.set_contacts(cs)
    pins = x0[o.pinned] + sc.h * sc.pin_velocity if o.pinned.size else None
    xo, _, info = o.frame(x0, v0, pin_targets=pins)
    thg = _parity.rows_from_triples(o, st["theta"])
    tho = info["theta_last"]
    d = np.flatnonzero(np.abs(thg - tho) > 1e-6 * np.maximum(1, np.abs(tho)))
    print(f"k={k}: err/tol {np.abs(xg - xo).max() / tol:.4g}  theta rows differing {d.size}"
          + (f" e.g. rows {d[:6].tolist()} gpu {thg[d[:6]].round(4).tolist()} oracle {tho[d[:6]].round(4).tolist()}"
             if d.size else ""), flush=True)

# local step at the oracle's own iterates x^k (sim_debug_local runs k_local on the given x)
o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=iters)
o.set_contacts(cs)
pins = x0[o.pinned] + sc.h * sc.pin_velocity if o.pinned.size else None
xo, _, info = o.frame(x0, v0, pin_targets=pins, capture=True)
h = sc.h
s_pred = x0 + h * v0 + h * h * np.asarray(sc.material.gravity)[None, :]
for k, rec in enumerate(info["iters"]):
    xk = rec["x_next"] if k == 0 else info["iters"][k - 1]["x_next"]
    xk = info["iters"][k - 1]["x_next"] if k > 0 else None
    if xk is None:
        continue
    Pg, rg = s.debug_local(xk, s_pred)
    F = O.deformation_gradients(xk, o.T, o.Bm)
    Po = O.project(F, o.model, o.k, o.mu, o.lam)
    _, sig, _ = O.signed_svd(F)
    err = np.linalg.norm(Pg - Po, axis=(1, 2)) / np.maximum(1.0, np.linalg.norm(Po, axis=(1, 2)))
    bad = np.flatnonzero(err > 1e-5)
    print(f"local at x^{k}: max rel err {err.max():.3g}, tets > 1e-5: {bad.size}, min sigma3 {sig[:, 2].min():.3g}, "
          f"min sigma3 of the bad ones {sig[bad, 2].min() if bad.size else float('nan'):.3g}, "
          f"inverted tets {int((sig[:, 2] < 0).sum())}", flush=True)
    ro = o.M[:, None] * (s_pred - xk) + O.elastic_forces(Po, F, o.Bm, o.w, o.h, o.T, o.n_v)
    print(f"   residual: max |r_gpu - r_oracle| / max |r_oracle| = "
          f"{np.abs(rg[o.free] - ro[o.free]).max() / np.abs(ro[o.free]).max():.3g}", flush=True)
