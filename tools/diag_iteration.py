"""One-iteration error of the GPU path inside a frame: for k = 1..iters-1, the oracle runs ONE
L-G iteration (Alg. 4 body) from the GPU's own iterate (x^k, lambda^k) -- the state
after a GPU frame of k iterations -- and is compared with the GPU's x^{k+1}.  Small one-step errors
with large frame errors mean the frame map amplifies rounding; a large one-step error means the
GPU computes a different iteration.  usage: python tools/diag_iteration.py <cfg5 instance> [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib

sc = scenes.make_scene("cfg3")
inst = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
v0, cs = scenes.batch_instance(sc, inst)
x0 = sc.mesh.X.copy()
tol = 1e-5 * sc.mesh.bbox_diag()
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_pin_velocity(sc.pin_velocity)
s.set_contacts(cs)
o = O.Oracle(sc.mesh, sc.material, sc.h)
o.set_contacts(cs)
h = sc.h
pins = x0[o.pinned] + h * sc.pin_velocity
spred = x0 + h * v0 + h * h * o.g[None, :]


def one_iteration(x, lam):
    """The body of Oracle.frame for one iteration from iterate x (pins already at target), lam."""
    F_ = o.free
    F = O.deformation_gradients(x, o.T, o.Bm)
    P = O.project(F, o.model, o.k, o.mu, o.lam)
    b = o.M[:, None] * spred + O.gt_p(P, o.Bm, o.w, h, o.T, o.n_v)
    b_f = b[F_] - o.A_fc @ x[o.pinned]
    theta, E, phi, Jx = o.indicators(x, x0, lam)
    kind = o.rows.kind
    xt = x.copy()
    xt[F_] = o.solve(b_f + h * h * o.JT(theta * lam)[F_])
    hvec = np.where(kind == 2, o.d_row - E * lam, np.where(kind == 0, -phi + theta * Jx, -h * phi + theta * Jx))
    rho = hvec - theta * o.Jx(xt)
    Cd = np.where(kind == 1, E / h, E / (h * h))
    z, _ = O.cr_solve(lambda v: theta * (o.D @ (theta * v)) + Cd * v, rho, o.cr_iters)
    lam = lam + z / (h * h)
    xn = x.copy()
    xn[F_] = o.solve(b_f + h * h * o.JT(theta * lam)[F_])
    return xn, lam


prev = None
for k in range(1, iters + 1):
    s.set_state(x0, v0)
    s.step(1, k)
    xg, _ = s.get_state()
    lg = s.get_lambda()
    if prev is not None:
        xo, lo = one_iteration(*prev)
        print(f"iteration {k}: one-step err/tol {np.abs(xg - xo).max() / tol:.4g}   "
              f"lambda rel {np.abs(lg - lo).max() / np.abs(lo).max():.3g}", flush=True)
    else:
        lam0 = np.zeros(o.m)
        xi = x0 + h * v0
        xi[o.pinned] = pins
        xo, lo = one_iteration(xi, lam0)
        print(f"iteration 1: one-step err/tol {np.abs(xg - xo).max() / tol:.4g}", flush=True)
    prev = (xg.copy(), lg.copy())

# the oracle's own frame, and the oracle continued from the GPU's iterate after k iterations
xi = x0 + h * v0
xi[o.pinned] = pins
st = (xi, np.zeros(o.m))
ref = []
for k in range(iters):
    st = one_iteration(*st)
    ref.append(st)
for k in range(1, iters):
    s.set_state(x0, v0)
    s.step(1, k)
    stg = (s.get_state()[0].copy(), s.get_lambda().copy())
    e0 = np.abs(stg[0] - ref[k - 1][0]).max() / tol
    for _ in range(k, iters):
        stg = one_iteration(*stg)
    print(f"oracle continued from the GPU's x^{k} (itself {e0:.3g} tol off the oracle's x^{k}): "
          f"frame end {np.abs(stg[0] - ref[-1][0]).max() / tol:.4g} tol off the oracle's frame", flush=True)
