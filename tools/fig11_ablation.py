"""Fig. 11 stick-slide ablation on the GPU: a stiff block
(rho = 1000, E = 1e8; cfg2, 10^3 vertices, 100 bottom contacts) on a 10-degree slope, 10 L-G
and 24 CR iterations, mu = mu* + delta with mu* = tan(10 deg) = 0.17632698.  For each
(NCP function, preconditioner) it reports the mean down-slope velocity after T seconds
against the rigid-limit closed form v = g (sin th - mu cos th) T (0 when mu >= mu*), and the
resolution: the smallest |delta| from which every larger |delta| is classified correctly
(slides: v >= 0.5 v_closed; sticks: v < 0.1 |v_closed(-delta)|).
Usage: python tools/fig11_ablation.py [frames]"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import scenes
import paper_2503_15078_b200 as simlib

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 100
th = 10.0
mus = math.tan(math.radians(th))
deltas = [0.1, 0.03, 0.01, 0.003, 0.001, 0.0005]
down = -np.array([math.cos(math.radians(th)), 0.0, math.sin(math.radians(th))])
torch.cuda.set_device(0)
out = {}
for ncp in (0, 1):
    for pre in (0, 1):
        rows = []
        for d in deltas:
            for sgn in (-1, 1):
                mu = mus + sgn * d
                sc = scenes.incline_block(theta_deg=th, mu=mu, nv=10, edge=0.1, youngs=1e8)
                sc.material.cr_iterations = 24
                s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
                s.set_ncp(ncp, pre)
                s.set_contacts(sc.contacts)
                s.step(frames, 10)
                x, v = s.get_state()
                vs = float((v @ down).mean())
                T = frames * sc.h
                vc = max(0.0, 9.81 * (math.sin(math.radians(th)) - mu * math.cos(math.radians(th))) * T)
                vslide = 9.81 * d * math.cos(math.radians(th)) * T      # |v_closed| at mu* - d
                ok = vs >= 0.5 * vc if sgn < 0 else abs(vs) < 0.1 * vslide
                rows.append({"delta": sgn * d, "mu": mu, "v": vs, "v_closed": vc, "ok": bool(ok)})
        res = None
        for d in sorted(deltas):
            if all(r["ok"] for r in rows if abs(r["delta"]) >= d - 1e-12):
                res = d
                break
        key = f"{'FB' if ncp == 0 else 'minmap'}+{'delassus' if pre == 0 else 'mass_inverse'}"
        out[key] = {"resolution": res, "rows": rows}
        print(key, "resolution", res, flush=True)
        for r in rows:
            print("   delta %+.4f  v %.3e  closed %.3e  %s" % (r["delta"], r["v"], r["v_closed"], "ok" if r["ok"] else "WRONG"))
json.dump({"frames": frames, "lg": 10, "cr": 24, "mu_star": mus, "results": out},
          open(os.path.join("gpurun_out", "fig11_ablation.json"), "w"), indent=1)
