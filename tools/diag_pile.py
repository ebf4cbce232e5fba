"""Grid CR vs cluster CR on the 9-cube pile (tests/test_gpu_grid_cr.py): re-synced frames; per L-G
iteration of each frame, the oracle's iteration from the GPU's own iterate vs the GPU's next iterate
(one-step err/tol), the indicators at that iterate (theta, C diagonal: sim_debug_contact_state of the
next iterate's frame) and the multipliers lambda^{k+1} (max relative difference)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib
from paper_2503_15078_b200._lib import debug_contact_state
import _parity

sc = scenes.pile(cells=3, nx=2, layers=2)
o = O.Oracle(sc.mesh, sc.material, sc.h)
o.set_contacts(sc.contacts)
tol = 1e-5 * sc.mesh.bbox_diag()
sims = {}
for mode in (1, 2):
    s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    s.set_cr_mode(mode)
    s.set_contacts(sc.contacts)
    sims[mode] = s
x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
for f in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    for mode, s in sims.items():
        its = _parity.gpu_iterates(s, x, v, 5)
        prev = None
        for k, (xg, lg) in enumerate(its):
            o.lg_iters = k + 1
            start = None if prev is None else (prev[0], prev[1], k)
            xo, _, info = o.frame(x, v, start=start, capture=True)
            o.lg_iters = 5
            s.set_state(x, v)
            s.step(1, k + 1)
            d = debug_contact_state(s)
            xs = x + sc.h * v + sc.h ** 2 * o.g[None, :] if prev is None else prev[0]
            ls = np.zeros(o.m) if prev is None else prev[1]
            th_o, E_o, _, _ = o.indicators(xs, x, ls)
            th_g = _parity.rows_from_triples(o, d["theta"])
            dth = float(np.abs(th_g - th_o).max())
            dl = float(np.abs(lg - info["lam"]).max() / max(1e-300, np.abs(info["lam"]).max()))
            e = np.abs(xg - xo).max() / tol
            extra = ""
            if e > 0.05 and prev is not None:   # the oracle's own one-step conditioning at this iterate
                sd = _parity.one_step_sensitivity(o, x, v, None, (prev[0], prev[1], k), k, tol)
                rng = np.random.default_rng(1)
                xp = prev[0] + 1e-7 * np.abs(prev[0]).max() * rng.standard_normal(prev[0].shape)
                o.lg_iters = k + 1
                xq, _, _ = o.frame(x, v, start=(xp, prev[1], k))
                o.lg_iters = 5
                rec = info["iters"][-1]
                hv_g = _parity.rows_from_triples(o, d["hvec"])
                dh = float(np.abs(hv_g - rec["theta"] * 0 - (rec["rho"] + rec["theta"] * o.Jx(rec["x_tilde"]))).max())
                dxt_o = (rec["x_tilde"] - prev[0])[d["slot_vertex"]]
                ddx = float(np.abs(d["dxt"] - dxt_o).max() / max(1e-300, np.abs(dxt_o).max()))
                extra = (f"; oracle one-step sensitivity: D noise {sd:.3g}, x noise 1e-7 {np.abs(xq - xo).max() / tol:.3g}"
                         f"; h-vector max diff {dh:.3g} (of {np.abs(hv_g).max():.3g}); dx~ at slots rel {ddx:.3g}")
            print(f"frame {f} mode {mode} iteration {k}->{k + 1}: one-step err/tol {e:.4g}, "
                  f"max|dtheta| {dth:.3g}, lambda rel {dl:.3g}{extra}", flush=True)
            prev = (xg, lg)
    # continue from the cluster-CR GPU state
    sims[1].set_state(x, v)
    sims[1].step(1, 5)
    x, v = sims[1].get_state()
