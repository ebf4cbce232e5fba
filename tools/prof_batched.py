"""Run a few batched cfg5 frames (S instances of cfg3) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib

S = int(sys.argv[1]) if len(sys.argv) > 1 else 128
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.cuda.set_device(0)
sc = scenes.make_scene("cfg3")
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_pin_velocity(sc.pin_velocity)
base = simlib.contacts_to_array(sc.contacts)
arrs, v0s = [], np.empty((S, sc.mesh.n_v, 3))
for i in range(S):
    v0s[i], d = scenes.batch_instance_params(sc, i)
    a = base.copy()
    a["offset"] += a["normal"][:, 2] * d
    arrs.append(a)
packed = (np.concatenate(arrs), np.full(S, len(base), np.int32))
s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), v0s)
for f in range(frames):
    s.set_contacts_batch(packed=packed)
    s.step(1, 5)
s.synchronize()
P = s.get_positions()
print("done", s.stats()["kernels_per_frame"], "finite", bool(np.isfinite(P).all()), "max|x-X|", float(np.abs(P - sc.mesh.X).max()))
