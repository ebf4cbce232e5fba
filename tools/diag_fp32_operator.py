"""Is a GPU-vs-oracle gap the fp32 representation of the sparse inverse, or a different
iteration?  For a scene small enough for dense algebra, the oracle's iteration is re-run with its
operators replaced by the GPU's: A^-1 by K32^T K32 and the Delassus D by J (K32^T K32) J^T, where K32
is the GPU's own fp32 K = L^-1 (sim_debug_get_inverse), evaluated in fp64.  If this oracle lands on
the GPU's iterates while the exact one does not, the gap is the fp32 storage of K (the method's
operator at fp32 resolution), not the arithmetic of the path.
usage: python tools/diag_fp32_operator.py [pile|mixed] [frames]"""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib
import _parity

which = sys.argv[1] if len(sys.argv) > 1 else "pile"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if which == "pile":
    sc = scenes.pile(cells=3, nx=2, layers=2)
    contacts = sc.contacts
else:
    import test_gpu_contact_kinds as T
    sc, cs = T._hanging_block(1e-6, offset=0.001)
    n = np.array([0.0, -math.sin(0.2), math.cos(0.2)])
    zmin = sc.mesh.X[:, 2].min()
    floor_pt = np.array([0.0, 0.0, zmin - 2e-4])
    bottom = np.flatnonzero(np.abs(sc.mesh.X[:, 2] - zmin) < 1e-12)
    t1, t2 = scenes.tangent_frame(n)
    contacts = []
    for k, v in enumerate(bottom):
        contacts.append(scenes.Contact([int(v)], [1.0], n, float(n @ floor_pt), mu=0.4, tangent1=t1, tangent2=t2))
        if k < len(cs):
            contacts.append(cs[k])
    contacts += cs[len(bottom):]
s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
s.set_contacts(contacts)
tol = 1e-5 * sc.mesh.bbox_diag()
ox = O.Oracle(sc.mesh, sc.material, sc.h)
ox.set_contacts(contacts)
o32 = O.Oracle(sc.mesh, sc.material, sc.h)
o32.set_contacts(contacts)
# the GPU's fp32 K in the oracle's free-vertex order
perm, parent, rowptr, vals = s.debug_inverse()
nf = perm.size
first = np.arange(nf) - np.diff(rowptr) + 1
K = np.zeros((nf, nf))
for i in range(nf):
    K[i, first[i]:i + 1] = vals[rowptr[i]:rowptr[i + 1]].astype(np.float64)
pos = {int(v): k for k, v in enumerate(o32.free)}
P = np.zeros((nf, nf))
for k in range(nf):
    P[k, pos[int(perm[k])]] = 1.0     # internal k <- oracle free index
Ainv32 = P.T @ (K.T @ K) @ P          # oracle free order
o32.solve = lambda b: Ainv32 @ b
# Delassus from the same operator (as set_contacts builds it from A_v^-1)
vc = o32.vc
idx = np.array([pos[int(v)] for v in vc])
G32 = Ainv32[np.ix_(idx, idx)]
o32.D = (o32.Wm @ G32 @ o32.Wm.T) * (o32.rows.c @ o32.rows.c.T)
print(f"# {which}: |D32 - D| / |D| = {np.abs(o32.D - ox.D).max() / np.abs(ox.D).max():.3g}", flush=True)
# the GPU's CR keeps theta and the C diagonal in fp32 shared memory: round them in the fp32 oracle
_ind = o32.indicators
def _ind32(x_, xt_, lam_):
    th, E, phi, Jx = _ind(x_, xt_, lam_)
    r32 = lambda a: np.asarray(a).astype(np.float32).astype(np.float64)
    kind = o32.rows.kind
    Cd = np.where(kind == 1, E / o32.h, E / (o32.h * o32.h))
    E32 = np.where(kind == 1, r32(Cd) * o32.h, r32(Cd) * o32.h * o32.h)
    return r32(th), E32, phi, Jx
o32.indicators = _ind32
x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
for f in range(frames):
    its = _parity.gpu_iterates(s, x, v, 5)
    prev = None
    for k, (xg, lg) in enumerate(its):
        start = None if prev is None else (prev[0], prev[1], k)
        res = []
        for o in (ox, o32):
            o.lg_iters = k + 1
            xo, _, _ = o.frame(x, v, start=start)
            o.lg_iters = 5
            res.append(np.abs(xg - xo).max() / tol)
        print(f"frame {f} iteration {k}->{k + 1}: GPU vs exact-operator oracle {res[0]:.4g} tol, vs fp32-K oracle {res[1]:.4g} tol",
              flush=True)
        prev = (xg, lg)
    s.set_state(x, v)
    s.step(1, 5)
    x, v = s.get_state()

# ---- isolate the CR: the GPU's own Schur RHS rho and step z = h^2 (lambda^{k+1} - lambda^k) at
# the iterate with the largest one-step gap, against the oracle's rho and its CR on the GPU's rho
from paper_2503_15078_b200._lib import debug_contact_rho, debug_contact_state
x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
worst = (0.0, None)
for f in range(frames):
    its = _parity.gpu_iterates(s, x, v, 5)
    prev = None
    for k, (xg, lg) in enumerate(its):
        start = None if prev is None else (prev[0], prev[1], k)
        ox.lg_iters = k + 1
        xo, _, info = ox.frame(x, v, start=start, capture=True)
        ox.lg_iters = 5
        e = np.abs(xg - xo).max() / tol
        if e > worst[0] and prev is not None:
            s.set_state(x, v)
            s.step(1, k + 1)
            ds = debug_contact_state(s)
            th_g = _parity.rows_from_triples(ox, ds["theta"])
            hv_g = _parity.rows_from_triples(ox, ds["hvec"])
            # the GPU's rho reconstructed from its h-vector and x~ = x^k + dxt at the slot vertices
            slot_of = {int(vv): q for q, vv in enumerate(ds["slot_vertex"])}
            xt_g = prev[0].copy()
            for vv, q in slot_of.items():
                xt_g[vv] = prev[0][vv] + ds["dxt"][q]
            rho_g = hv_g - th_g * ox.Jx(xt_g)
            xt_o = info["iters"][-1]["x_tilde"]
            dd = np.array([np.abs(xt_g[vv] - xt_o[vv]).max() for vv in slot_of])
            dref = np.array([np.abs(xt_o[vv] - prev[0][vv]).max() for vv in slot_of])
            qw = int(np.argmax(dd / np.maximum(dref, 1e-30)))
            rec = info["iters"][-1]
            kind = ox.rows.kind
            Cd = np.where(kind == 1, rec["E"] / ox.h, rec["E"] / (ox.h * ox.h))
            Sop = lambda q: rec["theta"] * (ox.D @ (rec["theta"] * q)) + Cd * q
            z_on_g, _ = O.cr_solve(Sop, rho_g, ox.cr_iters)
            z_g = (lg - prev[1]) * ox.h * ox.h
            z_o = rec["z"]
            worst = (e, f"frame {f} iteration {k}->{k + 1}: one-step {e:.3g} tol; |rho_gpu - rho_oracle| / |rho| = "
                        f"{np.abs(rho_g - rec['rho']).max() / np.abs(rec['rho']).max():.3g}; oracle CR on the GPU's rho vs "
                        f"GPU z: {np.abs(z_on_g - z_g).max() / np.abs(z_g).max():.3g}; oracle z vs GPU z: "
                        f"{np.abs(z_o - z_g).max() / np.abs(z_g).max():.3g}; max|dtheta| {np.abs(th_g - rec['theta']).max():.3g}; "
                        f"x~ at slots: max |gpu - oracle| {dd.max():.3g} m (worst rel. to its step {dd[qw] / max(dref[qw], 1e-30):.3g}, "
                        f"slot vertex {list(slot_of)[qw]})")
        prev = (xg, lg)
    s.set_state(x, v)
    s.step(1, 5)
    x, v = s.get_state()
print("# worst:", worst[1], flush=True)
