"""Dump the GPU's iterate after k L-G iterations of one cfg5 instance (n_instances = 1) to
gpurun_out/iter_<inst>_<k>.npz (x, v, lambda), for host-side analysis with the oracle.
usage: python tools/dump_iterate.py <instance> <k> [<k> ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import scenes
import paper_2503_15078_b200 as simlib

sc = scenes.make_scene("cfg3")
inst = int(sys.argv[1])
v0, cs = scenes.batch_instance(sc, inst)
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_pin_velocity(sc.pin_velocity)
s.set_contacts(cs)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
for k in map(int, sys.argv[2:]):
    s.set_state(sc.mesh.X, v0)
    s.step(1, k)
    x, v = s.get_state()
    np.savez(os.path.join(ROOT, "gpurun_out", f"iter_{inst}_{k}.npz"), x=x, v=v, lam=s.get_lambda())
print("ok")
