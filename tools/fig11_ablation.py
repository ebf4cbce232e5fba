"""Fig. 11 stick-slide ablation: a stiff block (rho = 1000, E = 1e8;
cfg2, 10^3 vertices, 100 bottom contacts) on a 10-degree slope, 10 L-G and 24 CR iterations,
mu = mu* + delta with mu* = tan(10 deg) = 0.17632698, T = frames * h.

GPU: for both frame-start readings (default A9/A10: x^0 = s, lambda^0 = 0; warm A9w/A10w:
x^0 = x_t + h v_t, lambda carried, sim_set_warm_start) and each (NCP function, preconditioner),
the mean down-slope velocity after T against the rigid-limit closed form
v = g (sin th - mu cos th) T (0 when mu >= mu*), and the resolution: the smallest |delta| from
which every larger |delta| is classified correctly (slides: v >= 0.5 v_closed; sticks:
v < 0.1 |v_closed(-delta)|).  Oracle (fp64, same readings, FB + Delassus): the same velocities at
delta = -+0.01, -+0.001 for comparison.
Usage: python tools/fig11_ablation.py [frames]"""
import json
import math
import os
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import scenes

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 100
th = 10.0
mus = math.tan(math.radians(th))
deltas = [0.1, 0.03, 0.01, 0.003, 0.001, 0.0005]
down = -np.array([math.cos(math.radians(th)), 0.0, math.sin(math.radians(th))])


def closed(mu):
    return max(0.0, 9.81 * (math.sin(math.radians(th)) - mu * math.cos(math.radians(th))) * frames * 0.01)


def oracle_run(args):
    warm, d = args
    from oracle import oracle as O
    sc = scenes.incline_block(theta_deg=th, mu=mus + d, nv=10, edge=0.1, youngs=1e8)
    o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=10, cr_iters=24, warm_start=warm)
    o.set_contacts(sc.contacts)
    x, v, lam = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X), None
    for _ in range(frames):
        x, v, info = o.frame(x, v, lam0=lam if warm else None)
        lam = info["lam"]
    return warm, d, float((v @ down).mean())


if __name__ == "__main__":
    import multiprocessing as mp
    jobs = [(w, s * d) for w in (False, True) for d in (0.01, 0.001) for s in (-1, 1)]
    pool = mp.get_context("fork").Pool(min(8, len(jobs)))
    pending = pool.map_async(oracle_run, jobs)          # CPU oracle runs while the GPU runs
    import torch
    import paper_2503_15078_b200 as simlib
    torch.cuda.set_device(0)
    out = {"frames": frames, "lg": 10, "cr": 24, "mu_star": mus, "results": {}}
    for warm in (False, True):
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
                        s.set_warm_start(warm)
                        s.set_contacts(sc.contacts)
                        s.step(frames, 10)
                        x, v = s.get_state()
                        s.close()
                        vs = float((v @ down).mean())
                        vc = closed(mu)
                        vslide = closed(mus - d)
                        ok = vs >= 0.5 * vc if sgn < 0 else abs(vs) < 0.1 * vslide
                        rows.append({"delta": sgn * d, "mu": mu, "v": vs, "v_closed": vc, "ok": bool(ok)})
                res = None
                for d in sorted(deltas):
                    if all(r["ok"] for r in rows if abs(r["delta"]) >= d - 1e-12):
                        res = d
                        break
                key = f"{'warm' if warm else 'default'}:{'FB' if ncp == 0 else 'minmap'}+" \
                      f"{'delassus' if pre == 0 else 'mass_inverse'}"
                out["results"][key] = {"resolution": res, "rows": rows}
                print(key, "resolution", res, flush=True)
                for r in rows:
                    print("   delta %+.4f  v %.3e  closed %.3e  %s" % (r["delta"], r["v"], r["v_closed"],
                                                                      "ok" if r["ok"] else "WRONG"), flush=True)
    orc = pending.get()
    out["oracle_fb_delassus"] = []
    print("oracle (fp64), FB + Delassus:")
    for warm, d, vo in orc:
        key = f"{'warm' if warm else 'default'}:FB+delassus"
        gv = next(r["v"] for r in out["results"][key]["rows"] if abs(r["delta"] - d) < 1e-12)
        out["oracle_fb_delassus"].append({"reading": "warm" if warm else "default", "delta": d, "v_oracle": vo,
                                          "v_gpu": gv})
        print("   %-7s delta %+.4f  v_oracle %.4e  v_gpu %.4e  closed %.3e" % ("warm" if warm else "default", d, vo,
                                                                               gv, closed(mus + d)))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "fig11_ablation.json"), "w"), indent=1)
