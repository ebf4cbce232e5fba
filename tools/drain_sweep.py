"""cfg5 frame time (S = 1024) and K-apply accuracy vs the TMEM fold interval (sim_set_kpass_mode)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib
from oracle import oracle as O
torch.cuda.set_device(0)
sc = scenes.make_scene("cfg3")
S = 1024
o = O.Oracle(sc.mesh, sc.material, sc.h)
rng = np.random.default_rng(3)
b = rng.standard_normal((sc.mesh.n_v, 3))
xo = o.solve(b[o.free])
for drain in (int(a) for a in (sys.argv[1:] or ["4", "8", "16", "1000"])):
    s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
    s.set_kpass_mode((drain << 4) | 2)
    s.set_pin_velocity(sc.pin_velocity)
    base = simlib.contacts_to_array(sc.contacts)
    arrs, v0s = [], np.empty((S, sc.mesh.n_v, 3))
    for i in range(S):
        v0s[i], d = scenes.batch_instance_params(sc, i)
        a = base.copy(); a["offset"] += a["normal"][:, 2] * d; arrs.append(a)
    packed = (np.concatenate(arrs), np.full(S, len(base), np.int32))
    s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), v0s)
    s.set_contacts_batch(packed=packed); s.step(2, 5); s.synchronize()
    t0 = time.perf_counter()
    for f in range(6):
        s.set_contacts_batch(packed=packed); s.step(1, 5)
    s.synchronize()
    ms = (time.perf_counter() - t0) / 6 * 1e3
    err = None
    try:
        xg = s.debug_apply_inverse(np.broadcast_to(b, (S,) + b.shape))
        err = float(max(np.abs(xg[i][o.free] - xo).max() for i in (0, 511, 1023)) / np.abs(xo).max())
    except Exception as e:
        err = repr(e)[:80]
    print(f"drain {drain}: {ms:.2f} ms/frame ({S * 5 / ms * 1e3:.0f} scene-iters/s wall), K-apply rel err {err}", flush=True)
    s.close()
