"""Single cfg3 scene: where the per-frame time goes when the contact set is re-committed every frame.
(a) events around commit + frame, (b) events around the frame only (commit before the start event),
(c) frames without a new commit; host-side seconds of the set_contacts and sim_step calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib

torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
sc = scenes.make_scene("cfg3")
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_stream(st.cuda_stream)
s.set_pin_velocity(sc.pin_velocity)
packed = s.pack_contacts(sc.contacts)
for _ in range(5):
    s.set_contacts(packed=packed)
    s.step(1, 5)
torch.cuda.synchronize()
N = 30
for mode in ("a", "b", "c"):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    th_set = th_step = 0.0
    for i in range(N):
        if mode == "a":
            ev[i][0].record(st)
        if mode != "c":
            t0 = time.perf_counter(); s.set_contacts(packed=packed); th_set += time.perf_counter() - t0
        if mode != "a":
            ev[i][0].record(st)
        t0 = time.perf_counter(); s.step(1, 5); th_step += time.perf_counter() - t0
        ev[i][1].record(st)
    torch.cuda.synchronize()
    ms = np.mean([a.elapsed_time(b) for a, b in ev])
    print(f"mode {mode}: {ms:.3f} ms per frame ({ms / 5:.4f} per L-G iteration); host set_contacts {1e3 * th_set / N:.3f} ms, "
          f"host sim_step {1e3 * th_step / N:.3f} ms per frame", flush=True)
