"""k_local device time per frame at S = 1024 for the three materials (Newton vs closed forms)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib
torch.cuda.set_device(0)
S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
for model in (0, 1, 2):
    sc = scenes.make_scene("cfg3")
    sc.material.model = model
    s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
    s.set_pin_velocity(sc.pin_velocity)
    s.step(2, 5)
    s.set_profiling(True)
    s.step(1, 5)
    s.step(1, 5)
    kt = s.kernel_times()
    print("model", model, "local ms/frame %.2f" % kt["local"], "gather %.2f" % kt["gather"], flush=True)
    s.close()
