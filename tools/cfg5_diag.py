"""Diagnose one cfg5 instance: GPU vs oracle lambda / contact classification after one frame."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib
inst = [int(a) for a in sys.argv[1:]] or [221]
sc = scenes.make_scene("cfg3")
S = 1024
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_pin_velocity(sc.pin_velocity)
base = simlib.contacts_to_array(sc.contacts)
arrs, v0s = [], np.empty((S, sc.mesh.n_v, 3))
for i in range(S):
    v0s[i], delta = scenes.batch_instance_params(sc, i)
    a = base.copy(); a["offset"] += a["normal"][:, 2] * delta; arrs.append(a)
s.set_contacts_batch(packed=(np.concatenate(arrs), np.full(S, len(base), np.int32)))
s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), v0s)
s.step(1, 5)
P = s.get_positions()
tol = 1e-5 * sc.mesh.bbox_diag()
for i in inst:
    v0, cs = scenes.batch_instance(sc, i)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    o.set_contacts(cs)
    pins = sc.mesh.X[o.pinned] + sc.h * sc.pin_velocity
    xo, _, info = o.frame(sc.mesh.X.copy(), v0s[i], pin_targets=pins)
    lo = info["lam"]; lg = s.get_lambda(i)
    x_t = sc.mesh.X
    co, cg = o.classify(xo, x_t, lo), o.classify(P[i], x_t, lg)
    err = np.abs(P[i] - xo).max(axis=1)
    worst = np.argsort(-err)[:5]
    print(f"inst {i}: err/tol {err.max()/tol:.3f}; classes oracle {np.bincount(co, minlength=3)} gpu {np.bincount(cg, minlength=3)}; differ {np.flatnonzero(co != cg)[:10]}")
    d = np.flatnonzero(co != cg)
    for c in d[:6]:
        j = 3 * c
        print(f"   contact {c} vert {cs[c].verts} oracle cls {co[c]} lam {lo[j:j+3]}  gpu cls {cg[c]} lam {lg[j:j+3]}")
    print("   worst verts", worst, err[worst] / tol, "contact verts near:", [c for c in range(len(cs)) if cs[c].verts[0] in worst][:5])
    print("   max |dlam_n|", np.abs(lo[0::3] - lg[0::3]).max(), "max lam_n", lo[0::3].max())
