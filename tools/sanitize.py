"""Small end-to-end runs for compute-sanitizer: single scene with contacts (cluster CR), grid CR,
batched instances on the tensor-core passes (S = 3 with ADMM, S = 80 with one CR CTA per
instance), proximity query, the 9-cube pile, cfg1 batched without contacts; round 2: the persistent
small-scene kernel, the plane tensor-core K-passes (S = 130, 5, 6), paired / scalar local steps,
a drop tolerance."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scenes
import paper_2503_15078_b200 as sl

sc = scenes.incline_block(theta_deg=10.0, mu=math.tan(math.radians(10.0)) - 0.05, nv=4, edge=0.1, youngs=1e7)
for mode in (1, 2):
    s = sl.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    s.set_cr_mode(mode)
    s.set_contacts(sc.contacts)
    s.step(2, 3)
    s.synchronize()
S = 3
s = sl.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_contacts_batch([sc.contacts] * S)
s.set_admm(True)
s.step(2, 3)
s.synchronize()
# S = 80: one CR CTA per instance (G_A gathered into shared memory, row-per-thread matvec),
# tensor-core chain / scatter passes split over tile ranges
S = 80
s = sl.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_contacts_batch([sc.contacts] * S)
s.step(2, 3)
s.synchronize()
s = sl.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.detect_contacts(sc.obstacles, np.arange(sc.mesh.n_v), 2e-3)
s.step(1, 3)
s.synchronize()
p = scenes.pile(cells=3, nx=2, layers=2)
s = sl.Sim(p.mesh.X, p.mesh.T, p.mesh.fixed, p.material, p.h)
s.set_contacts(p.contacts)
s.step(1, 3)
s.synchronize()
g = scenes.make_scene("cfg1")
s = sl.Sim(g.mesh.X, g.mesh.T, g.mesh.fixed, g.material, g.h, n_instances=4)
s.step(1, 2)
s.synchronize()
# round 2: the persistent small-scene kernel (cfg1, one instance), the plane tensor-core K-passes
# with a partial second chunk and odd S (Sp padding, scalar local step) and even S (paired local
# step), the CUDA-core batched passes, a drop tolerance
s = sl.Sim(g.mesh.X, g.mesh.T, g.mesh.fixed, g.material, g.h)
s.step(3, 5)
s.synchronize()
b = scenes.make_scene("block", nv=5)
for S, mode in ((130, 2), (5, 2), (6, 1)):
    s = sl.Sim(b.mesh.X, b.mesh.T, b.mesh.fixed, b.material, b.h, n_instances=S, drop_tolerance=1e-3 if S == 6 else 0.0)
    s.set_kpass_mode(mode)
    s.set_contacts_batch([[]] * S)
    s.step(2, 3)
    s.synchronize()
s = sl.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=130)
s.set_contacts_batch([sc.contacts] * 130)
s.step(1, 3)
s.synchronize()
print("sanitize run done")
