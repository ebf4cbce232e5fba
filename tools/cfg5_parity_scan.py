"""cfg5 parity scan: one frame (5 L-G / 10 CR) of the 1024 cfg5 instances (SURVEY §8(d) cfg5:
initial velocity N(0, 0.01^2) m/s, obstacle offset U(-5, +5) mm) on the GPU, against the fp64
oracle on sampled instances: every `stride`-th instance plus the `deep` deepest initial
penetrations.  Per instance and GPU variant: err/tol = max |x_gpu - x_oracle| / (1e-5 bbox),
and whether the frame-end classification (A21, outside the exclusion band) is identical.

Variants (--modes, comma separated):
  ts     batched tensor-core K-passes (the default product path, sim_set_kpass_mode 2)
  ts2    the same with an fp64 fold of the TMEM accumulators every 2 tiles
  core   batched CUDA-core FP32 K-passes (sim_set_kpass_mode 1)
  tscc   tensor-core K-passes with CUDA-core contact chain / scatter passes (sim_set_kpass_mode 3)
  single the instance alone (n_instances = 1: HBM-streaming SpMV path), only for --single-max
         instances (the deepest first)

usage: python tools/cfg5_parity_scan.py [--stride 64] [--deep 32] [--modes ts,core,single]
       [--out profiles/x.txt]
"""
import argparse
import os
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib
import _parity

ap = argparse.ArgumentParser()
ap.add_argument("--stride", type=int, default=64)
ap.add_argument("--deep", type=int, default=32)
ap.add_argument("--modes", default="ts,core,single")
ap.add_argument("--single-max", type=int, default=16)
ap.add_argument("--out", default=None)
a = ap.parse_args()
modes = a.modes.split(",")

sc = scenes.make_scene("cfg3")
S = 1024
tol = 1e-5 * sc.mesh.bbox_diag()
base = simlib.contacts_to_array(sc.contacts)
v0s = np.empty((S, sc.mesh.n_v, 3))
deltas = np.empty(S)
arrs = []
for i in range(S):
    v0s[i], deltas[i] = scenes.batch_instance_params(sc, i)
    ar = base.copy()
    ar["offset"] += ar["normal"][:, 2] * deltas[i]
    arrs.append(ar)
packed = (np.concatenate(arrs), np.full(S, len(base), np.int32))
X0 = np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape)
sel = list(range(0, S, a.stride))
deep = [int(c) for c in np.argsort(-deltas)[:a.deep]]
sel += [c for c in deep if c not in sel]

gpu = {}
lam_g = {}
kp = {"ts": 2, "ts2": (2 << 4) | 2, "core": 1, "tscc": 3}
s = None
for m in modes:
    if m == "single":
        continue
    for iters in (1, 5):
        t0 = time.time()
        if s is None:
            s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
            s.set_pin_velocity(sc.pin_velocity)
        s.set_kpass_mode(kp[m])
        s.set_contacts_batch(packed=packed)
        s.set_states(X0, v0s)           # lambda restarts from 0 as well
        s.step(1, iters)
        gpu[(m, iters)] = {i: p for i, p in enumerate(s.get_positions()) if i in sel}
        lam_g[(m, iters)] = {i: s.get_lambda(i) for i in sel}
        print(f"# GPU {m} {iters} iteration(s): {time.time() - t0:.1f}s", flush=True)
if s is not None:
    s.close()
if "single" in modes:
    s1 = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    s1.set_pin_velocity(sc.pin_velocity)
    for iters in (1, 5):
        gpu[("single", iters)], lam_g[("single", iters)] = {}, {}
        for i in deep[:a.single_max]:
            _, cs = scenes.batch_instance(sc, i)
            s1.set_contacts(cs)
            s1.set_state(sc.mesh.X, v0s[i])
            s1.step(1, iters)
            gpu[("single", iters)][i] = s1.get_state()[0]
            lam_g[("single", iters)][i] = s1.get_lambda()
    s1.close()


def oracle_instance(i):
    """fp64 oracle frames (1 and 5 L-G iterations) of instance i against every GPU variant."""
    t0 = time.time()
    v0, cs = scenes.batch_instance(sc, i)
    res = {}
    for iters in (1, 5):
        o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=iters)
        o.set_contacts(cs)
        pins = sc.mesh.X[o.pinned] + sc.h * sc.pin_velocity
        xo, _, info = o.frame(sc.mesh.X.copy(), v0s[i], pin_targets=pins)
        sens = None
        for (m, it), d in gpu.items():
            if it != iters or i not in d:
                continue
            e = float(np.abs(d[i] - xo).max()) / tol
            bad, n = _parity.classification_mismatches(o, d[i], sc.mesh.X, lam_g[(m, it)][i], xo, info["lam"], tol)
            if e > 1.0 and sens is None:   # the frame's own conditioning (tests/_parity.py frame_sensitivity)
                sens = _parity.frame_sensitivity(o, sc.mesh.X.copy(), v0s[i], tol, pins)
            res[(m, it)] = (e, bad, n, sens if e > 1.0 else None)
    return i, res, time.time() - t0


if __name__ == "__main__":
    import multiprocessing as mp
    nproc = int(os.environ.get("SCAN_PROCS", str(max(1, min(16, (os.cpu_count() or 2) // 2)))))
    with mp.get_context("fork").Pool(nproc) as pool:
        results = pool.map(oracle_instance, sel)
    lines = [f"# tools/cfg5_parity_scan.py --stride {a.stride} --deep {a.deep} --modes {a.modes}: 1024 cfg5 "
             f"instances (v0 ~ N(0, 0.01^2) m/s, obstacle offset delta ~ U(-5,+5) mm, positive = penetrating start), "
             f"one frame of 1 and of 5 L-G iterations; err/tol = max|x_gpu - x_oracle| / (1e-5 bbox); cls = "
             f"frame-end classification mismatches outside the tolerance band / contacts compared"]
    worst = {}
    for i, res, dt in results:
        pen = deltas[i] > 0
        parts = []
        for (m, it), (e, bad, n, sens) in sorted(res.items()):
            key = (m, it, "penetrating" if pen else "non-penetrating")
            w = worst.setdefault(key, [0.0, 0, 0, 0])
            w[0] = max(w[0], e)
            w[1] += bad
            w[2] += e > 1.0
            guard = 1.0 if sens is None or sens < _parity.WELL_CONDITIONED else max(_parity.ILL_GUARD, 2.0 * sens)
            w[3] += e > guard
            parts.append(f"{m}/{it} {e:8.3f} cls {bad}/{n}" + (f" (sens {sens:.3f}, guard {guard:.2f})" if sens is not None else ""))
        ln = f"inst {i:4d} delta {deltas[i] * 1e3:+.2f} mm  " + "  ".join(parts) + f"  ({dt:.1f}s)"
        print(ln, flush=True)
        lines.append(ln)
    for (m, it, kind), (w, bad, over, over_guard) in sorted(worst.items()):
        lines.append(f"# {m}, {it} iteration(s), {kind}: worst err/tol {w:.3f}, instances over tol {over} "
                     f"(over the conditioning guard of tests/_parity.py: {over_guard}), classification mismatches {bad}")
        print(lines[-1])
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")
