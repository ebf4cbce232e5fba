"""Tensor-core batched K-pass vs CUDA-core FP32 and the oracle (apply-inverse), then timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib

torch.cuda.set_device(0)
for name, S in (("block", 33), ("cfg3", 130)):
    sc = scenes.make_scene(name, **({"nv": 7, "split": "kuhn6"} if name == "block" else {}))
    s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    rng = np.random.default_rng(5)
    b = rng.standard_normal((S, sc.mesh.n_v, 3)).astype(np.float32).astype(np.float64)
    res = {}
    modes = (1, 64, 66, 130)
    for mode in modes:
        s.set_kpass_mode(mode)
        res[mode] = s.debug_apply_inverse(b)
    errs = []
    for i in (0, 1, S // 2, S - 1):
        xr = o.solve(b[i][o.free])
        errs.append([np.abs(res[m][i][o.free] - xr).max() / np.abs(xr).max() for m in modes])
    print(name, S, "rel err vs oracle, modes", modes, np.array(errs).max(0), flush=True)
# timing at S = 1024 frames (both modes)
sc = scenes.make_scene("cfg3")
S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_pin_velocity(sc.pin_velocity)
base = simlib.contacts_to_array(sc.contacts)
packed = (np.concatenate([base] * S), np.full(S, len(base), np.int32))
s.set_contacts_batch(packed=packed)
for mode in (1, 64, 66, 130):
    s.set_kpass_mode(mode)
    s.step(1, 5)
    s.set_profiling(True)
    s.step(1, 5)
    s.step(1, 5)
    kt = s.kernel_times()
    s.set_profiling(False)
    print("mode", mode, "S", S, {k: round(v, 2) for k, v in kt.items()}, flush=True)
x = s.get_positions()
print("finite", np.isfinite(x).all())
