"""cfg3 single scene (S = 1): device ms per frame with and without in-graph kernel events,
per-kernel breakdown.  Usage: python tools/prof_single.py [frames]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 20
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
sc = scenes.make_scene("cfg3")
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_stream(st.cuda_stream)
s.set_pin_velocity(sc.pin_velocity)
packed = s.pack_contacts(sc.contacts)
for mode in ("reset", "keep"):
    for _ in range(5):
        s.set_contacts(packed=packed)
        s.step(1, 5)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(frames + 1)]
    ev[0].record(st)
    for f in range(frames):
        if mode == "reset":
            s.set_contacts(packed=packed)
        s.step(1, 5)
        ev[f + 1].record(st)
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(frames)]
    print(mode, "frame ms median %.3f min %.3f -> %.4f ms per L-G iteration" % (np.median(ms), min(ms), np.median(ms) / 5))
s.set_profiling(True)
s.step(1, 5)
kt = {k: 0.0 for k in simlib.KERNEL_KINDS}
for f in range(5):
    s.step(1, 5)
    for k, v in s.kernel_times().items():
        kt[k] += v / 5
print("per-frame kernel us (in-graph events, serialised):", {k: round(1000 * v, 1) for k, v in kt.items()},
      "sum %.1f" % (1000 * sum(kt.values())))
print(s.stats())
