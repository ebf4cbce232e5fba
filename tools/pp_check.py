"""TS K-passes, ping-pong accumulators (kpass mode 3) vs mode 2: K-apply accuracy against the
oracle's sparse LU and cfg5 frame time at S = 1024."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib
from oracle import oracle as O
torch.cuda.set_device(0)
sc = scenes.make_scene("cfg3")
o = O.Oracle(sc.mesh, sc.material, sc.h)
rng = np.random.default_rng(3)
for S in (200, 1024):
    b = rng.standard_normal((S, sc.mesh.n_v, 3))
    for mode in (2, 3):
        s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
        s.set_kpass_mode(mode)
        xg = s.debug_apply_inverse(b)
        errs = []
        for i in (0, S // 2, S - 1):
            xo = o.solve(b[i][o.free])
            errs.append(np.abs(xg[i][o.free] - xo).max() / np.abs(xo).max())
        line = f"S {S} mode {mode}: K-apply rel err {max(errs):.2e}"
        if S == 1024:
            s.set_pin_velocity(sc.pin_velocity)
            base = simlib.contacts_to_array(sc.contacts)
            arrs, v0s = [], np.empty((S, sc.mesh.n_v, 3))
            for i in range(S):
                v0s[i], d = scenes.batch_instance_params(sc, i)
                a = base.copy(); a["offset"] += a["normal"][:, 2] * d; arrs.append(a)
            packed = (np.concatenate(arrs), np.full(S, len(base), np.int32))
            s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), v0s)
            s.set_contacts_batch(packed=packed); s.step(2, 5); s.synchronize()
            s.set_profiling(True)
            s.set_contacts_batch(packed=packed); s.step(1, 5)
            kt = s.kernel_times()
            line += f"; kpass1 {kt['kpass1']:.2f} ms/frame, kpass2 {kt['kpass2']:.2f} ms/frame"
            P = s.get_positions()
            line += f"; finite {bool(np.isfinite(P).all())}"
        print(line, flush=True)
        s.close()
