"""Phase timeline of the cluster CR on the single cfg3 scene (sim_debug_cr_timeline, %globaltimer ns):
staging, first reduction, each CR iteration, and inside iteration 3: W (J^T Theta v per active
slot), the G_A matvec with the cluster exchange, the reduction + vector update."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scenes
import paper_2503_15078_b200 as simlib
from paper_2503_15078_b200._lib import debug_cr_timeline

sc = scenes.make_scene("cfg3")
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_pin_velocity(sc.pin_velocity)
s.set_contacts(sc.contacts)
s.step(3, 5)
s.synchronize()
t = debug_cr_timeline(s)
print("raw (us from the CR kernel start):", np.round(t[:24], 2).tolist())
print("staging %.2f us, first reduction %.2f us" % (t[1] - t[0], t[2] - t[1]))
its = [t[3 + i] - (t[2] if i == 0 else t[3 + i - 1]) for i in range(9) if i != 3]
print("CR iterations (us):", np.round(its, 2).tolist())
print("iteration 3: W %.2f us, matvec + exchange %.2f us, reduction + update %.2f us" % (t[13] - t[12], t[16] - t[13], t[17] - t[16]))
print("epilogue %.2f us; active slots %d, G_A in smem %d, cluster %d" % (t[21] - t[20], (t[31] - t[0]) / 1000, int((t[30] - t[0]) / 1000) % 10, int((t[30] - t[0]) / 10000)))
print("staging: active list %.2f, G_A copies issued %.2f, rho/vectors %.2f, copies landed %.2f, cluster sync %.2f us"
      % (t[22] - t[0], t[23] - t[22], t[24] - t[23], t[25] - t[24], t[1] - t[25]))
