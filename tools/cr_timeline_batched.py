"""CR phase timeline (instance 0) at S instances (one CTA per instance when S >= 148)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib
from paper_2503_15078_b200._lib import debug_cr_timeline
S = int(sys.argv[1]) if len(sys.argv) > 1 else 128
torch.cuda.set_device(0)
sc = scenes.make_scene("cfg3")
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_pin_velocity(sc.pin_velocity)
base = simlib.contacts_to_array(sc.contacts)
s.set_contacts_batch(packed=(np.concatenate([base] * S), np.full(S, len(base), np.int32)))
for f in range(3):
    s.step(1, 5)
s.synchronize()
tl = debug_cr_timeline(s)
print("S", S, "CR timeline us:", " ".join(f"{v:.1f}" for v in tl[:12]), "| it3: start %.1f W %.1f mv %.1f wait %.1f Sv %.1f end %.1f" % tuple(tl[12:18]), "| end", f"{tl[20]:.1f} {tl[21]:.1f}", "na", int(tl[31]), "gA_smem+10*csize", tl[30])
