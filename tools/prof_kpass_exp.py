"""cfg5 (S = 1024) per-frame kernel times from in-graph events, frames restarted from the cfg5 initial states (K-pass A/B runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib
torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
sc = scenes.make_scene("cfg3")
S = 1024
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_stream(st.cuda_stream)
s.set_pin_velocity(sc.pin_velocity)
base = simlib.contacts_to_array(sc.contacts)
arrs, v0s = [], np.empty((S, sc.mesh.n_v, 3))
for i in range(S):
    v0s[i], d = scenes.batch_instance_params(sc, i)
    a = base.copy(); a["offset"] += a["normal"][:, 2] * d; arrs.append(a)
packed = (np.concatenate(arrs), np.full(S, len(base), np.int32))
s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), v0s)
s.set_contacts_batch(packed=packed)
s.step(1, 5)
s.set_profiling(True)
kt = {k: 0.0 for k in simlib.KERNEL_KINDS}
for f in range(3):
    s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), v0s)
    s.step(1, 5)
    for k, v in s.kernel_times().items():
        kt[k] += v / 3
print({k: round(v, 3) for k, v in kt.items()})
print("kpass1 %.3f kpass2 %.3f ms per frame" % (kt["kpass1"], kt["kpass2"]))
