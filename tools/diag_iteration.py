"""Where a GPU frame departs from the oracle's (cfg5 instance, default readings A9/A10:
x^0 = s, lambda^0 = 0).  For k = 0..iters-1 the GPU's iterate (x^k, lambda^k) is taken from a
GPU frame of k iterations, then
  * local: the GPU's projections P (sim_debug_local, fp32) vs the oracle's at the same x^k
    (max |P_gpu - P_oracle|_F / max(1, |P_oracle|_F), the worst tets' smallest singular values);
  * one-step: the oracle runs ONE L-G iteration (Alg. 4 body) from the GPU's
    (x^k, lambda^k), compared with the GPU's x^{k+1}; "with P_gpu" repeats it with the GPU's
    projections, isolating the global / contact part.
Small one-step errors with a large frame error mean the frame map amplifies rounding; a large
one-step error means the GPU computes a different iteration.
With --batch S the GPU runs S copies of the instance in one handle (the batched path) and
instance 0 is compared.
usage: python tools/diag_iteration.py <cfg5 instance> [iters] [--batch S]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib

sc = scenes.make_scene("cfg3")
args = [a for a in sys.argv[1:] if not a.startswith("--")]
inst = int(args[0])
iters = int(args[1]) if len(args) > 1 else 5
S = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 1
if S > 1:
    args = [a for a in args if a != str(S)] if len(args) > 2 else args
v0, cs = scenes.batch_instance(sc, inst)
x0 = sc.mesh.X.copy()
tol = 1e-5 * sc.mesh.bbox_diag()
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)
s.set_pin_velocity(sc.pin_velocity)
if S > 1:
    s.set_contacts_batch([cs] * S)
else:
    s.set_contacts(cs)
o = O.Oracle(sc.mesh, sc.material, sc.h)
o.set_contacts(cs)
h = sc.h
pins = x0[o.pinned] + h * sc.pin_velocity
spred = x0 + h * v0 + h * h * o.g[None, :]


def one_iteration(x, lam, P=None):
    F_ = o.free
    F = O.deformation_gradients(x, o.T, o.Bm)
    if P is None:
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
    return xn, lam, E


xi = spred.copy()
xi[o.pinned] = pins
gpu = [(xi, np.zeros(o.m))]
for k in range(1, iters + 1):
    for i in range(S):
        s.set_state(x0, v0, instance=i)
    s.step(1, k)
    gpu.append((s.get_state()[0].copy(), s.get_lambda().copy()))
for k in range(iters):
    xk, lk = gpu[k]
    F = O.deformation_gradients(xk, o.T, o.Bm)
    Po = O.project(F, o.model, o.k, o.mu, o.lam)
    Pg = s.debug_local(xk, spred)[0].astype(np.float64) if S == 1 else Po
    dP = np.linalg.norm(Pg - Po, axis=(1, 2)) / np.maximum(1.0, np.linalg.norm(Po, axis=(1, 2)))
    worst = np.argsort(-dP)[:3]
    sig = np.linalg.svd(F[worst], compute_uv=False)
    xo, lo, E = one_iteration(xk, lk)
    xp, _, _ = one_iteration(xk, lk, P=Pg)
    xg1, lg1 = gpu[k + 1]
    print(f"iteration {k}->{k + 1}: local max dP {dP.max():.3g} (tets {list(worst)}, sigma {np.round(sig, 4).tolist()}); "
          f"one-step err/tol {np.abs(xg1 - xo).max() / tol:.4g}, with P_gpu {np.abs(xg1 - xp).max() / tol:.4g}; "
          f"lambda rel {np.abs(lg1 - lo).max() / np.abs(lo).max():.3g}; max E_f {E[1::3].max():.3g}", flush=True)

xo_frame, _, _ = o.frame(x0, v0, pin_targets=pins)
print(f"frame ({iters} iterations, S = {S}): GPU vs oracle {np.abs(gpu[-1][0] - xo_frame).max() / tol:.4g} tol", flush=True)
