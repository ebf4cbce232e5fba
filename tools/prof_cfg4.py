"""cfg4 (multi-object pile, ~1M DoF, ~18k contacts): frame time, per-kernel breakdown,
K-pass GB/s.  Usage: python tools/prof_cfg4.py [frames]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 10
torch.cuda.set_device(0)
t0 = time.time()
sc = scenes.make_scene("cfg4")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_stream(st.cuda_stream)
packed = s.pack_contacts(sc.contacts)
s.set_contacts(packed=packed)
print("setup s", round(time.time() - t0, 1), "build s", round(s.stats()["build_seconds"], 1), flush=True)
for _ in range(3):
    s.set_contacts(packed=packed)
    s.step(1, 5)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(frames + 1)]
ev[0].record(st)
for f in range(frames):
    s.set_contacts(packed=packed)
    s.step(1, 5)
    ev[f + 1].record(st)
torch.cuda.synchronize()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(frames)]
st_ = s.stats()
print("frame ms median %.3f  per L-G iteration %.3f ms" % (np.median(ms), np.median(ms) / 5))
print({k: st_[k] for k in ("n_vertices", "n_tets", "nnz_K", "etree_height", "n_contacts", "n_contact_vertices",
                            "kernels_per_frame", "last_cr_residual", "n_active", "max_abs_phi_n")})
s.set_profiling(True)
s.step(1, 5)
tot = {k: 0.0 for k in simlib.KERNEL_KINDS}
for f in range(3):
    s.step(1, 5)
    kt = s.kernel_times()
    for k in tot:
        tot[k] += kt[k] / 3
s.set_profiling(False)
print("per-frame kernel ms:", {k: round(v, 3) for k, v in tot.items()})
nnz, nf = st_["nnz_K"], st_["n_free"]
for k in ("kpass1", "kpass2"):
    us = tot[k] / 5 * 1e3
    print(k, "us/launch %.1f" % us, "GB/s %.0f" % ((4 * nnz + 48 * nf) / (us * 1e-6) / 1e9))
x, v = s.get_state()
print("min z", x[:, 2].min(), "max|v|", np.abs(v).max(), "finite", np.isfinite(x).all())
