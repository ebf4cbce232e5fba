"""Compare one L-G iteration's contact intermediates GPU vs oracle on cfg3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib
from paper_2503_15078_b200._lib import debug_contact_state

torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sc = scenes.make_scene(name) if name != "incline" else scenes.incline_block(theta_deg=10, mu=0.23, nv=5, edge=0.1, youngs=1e8)
x0, v0 = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
pins = x0[sc.mesh.fixed.astype(bool)] + sc.h * sc.pin_velocity
o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=1)
o.set_contacts(sc.contacts)
xo, _, info = o.frame(x0, v0, pin_targets=pins, capture=True)
rec = info["iters"][0]
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_pin_velocity(sc.pin_velocity)
s.set_contacts(sc.contacts)
s.step(1, 1)
xg, _ = s.get_state()
lg = s.get_lambda()
cs = debug_contact_state(s)
h = sc.h
print("D_jj rel", np.abs(cs["djj"] - np.diag(o.D)[0::3]).max() / np.abs(np.diag(o.D)).max())
print("theta max diff", np.abs(cs["theta"] - rec["theta"]).max())
kind = o.rows.kind
Cor = np.where(kind == 1, rec["E"] / h, rec["E"] / (h * h))
print("C rel", np.abs(cs["cdiag"] - Cor).max() / np.abs(Cor).max())
Jx = o.Jx(x0 if False else xo * 0 + info["iters"][0]["x_tilde"] * 0 + x0)  # placeholder
# oracle x~ - x at slot vertices
xt_or = rec["x_tilde"]
s_v = cs["slot_vertex"]
# x^0 = s for free vertices
s_pred = x0 + h * v0 + h * h * np.asarray(sc.material.gravity)
dx_or = xt_or[s_v] - s_pred[s_v]
print("dxt rel", np.abs(cs["dxt"] - dx_or).max() / np.abs(dx_or).max(), "max", np.abs(dx_or).max())
# rho from hvec
hv_or = np.where(kind == 2, 0, 0)  # recompute oracle hvec
theta, E, phi, Jx = rec["theta"], rec["E"], rec["phi"], None
print("lam rel", np.abs(lg - info["lam"]).max() / np.abs(info["lam"]).max())
z_or = rec["z"]; z_g = lg * h * h
print("z rel", np.abs(z_g - z_or).max() / np.abs(z_or).max())
print("x max diff", np.abs(xg - xo).max())
# rho check via oracle pieces
rho = rec["rho"]
print("rho max", np.abs(rho).max())
xtg = s_pred.copy()
xtg[o.pinned] = pins
xtg[s_v] += cs["dxt"]
rho_g = cs["hvec"] - cs["theta"] * o.Jx(xtg)
print("rho rel", np.abs(rho_g - rho).max() / np.abs(rho).max())
i = np.argmax(np.abs(rho_g - rho)); print(" worst row", i, rho_g[i], rho[i], "theta", cs["theta"][i], theta[i])
# CR on oracle matrix with GPU rho
S = lambda v: theta * (o.D @ (theta * v)) + Cor * v
zz, _ = O.cr_solve(S, rho_g, o.cr_iters)
print("oracle CR on gpu rho vs gpu z rel", np.abs(zz - z_g).max() / np.abs(z_g).max())
