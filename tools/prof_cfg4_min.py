"""cfg4: setup + `frames` frames, nothing else (for ncu launch lists / captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenes
import paper_2503_15078_b200 as simlib

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
torch.cuda.set_device(0)
sc = scenes.make_scene("cfg4")
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
packed = s.pack_contacts(sc.contacts)
for f in range(frames):
    s.set_contacts(packed=packed)
    s.step(1, 5)
s.synchronize()
print("done", s.stats()["kernels_per_frame"])
