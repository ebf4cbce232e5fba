"""Drop tolerance (reading A25): for tol in {0, 1e-4, 1e-3}, the host build time,
the K entries kept, the bytes one K-pass pair streams (sim_stats.kpass_bytes), the fraction of the
32-row x 32-column K tiles that keep at least one entry (what skipping empty tiles could save), and
the error of the GPU's K^T K b against the oracle's exact sparse-LU solve of A_v x = b (random b),
max-relative.
usage: python tools/drop_tolerance.py [cfg3|cfg4] [n_instances]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import scenes
from oracle import oracle as O
import paper_2503_15078_b200 as simlib

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sc = scenes.make_scene(name)
o = O.Oracle(sc.mesh, sc.material, sc.h)
rng = np.random.default_rng(3)
b = rng.standard_normal((S, sc.mesh.n_v, 3)).astype(np.float32).astype(np.float64)
xr = [o.solve(b[i][o.free]) for i in range(S)]
print(f"# {name}: {sc.mesh.n_v} v / {sc.mesh.n_t} t, n_instances = {S}", flush=True)
for tol in (0.0, 1e-4, 1e-3):
    t0 = time.time()
    s = simlib.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, drop_tolerance=tol, n_instances=S)
    tb = time.time() - t0
    st = s.stats()
    perm, parent, rowptr, vals = s.debug_inverse()
    n = len(parent)
    first = np.arange(n) - np.diff(rowptr) + 1
    tiles = kept_tiles = 0
    for b0 in range(0, n, 32):
        b1 = min(n, b0 + 32)
        c0 = int(first[b0:b1].min())
        anyt = np.zeros((b1 - c0 + 31) // 32, bool)
        occ = np.zeros_like(anyt)
        for i in range(b0, b1):
            t = (np.arange(first[i], i + 1) - c0) // 32
            anyt[t] = True
            occ[t[vals[rowptr[i]:rowptr[i + 1]] != 0]] = True
        tiles += int(anyt.sum())
        kept_tiles += int(occ.sum())
    x = s.debug_apply_inverse(b if S > 1 else b[0])
    x = x.reshape(S, sc.mesh.n_v, 3)
    err = max(float(np.abs(x[i][o.free] - xr[i]).max() / np.abs(xr[i]).max()) for i in range(S))
    print(f"tol {tol:g}: build {tb:.2f} s (phases {[round(q, 3) for q in st['build_phase_seconds']]}), nnz(K) {st['nnz_K']} "
          f"kept {st['nnz_K_kept']} ({st['nnz_K_kept'] / st['nnz_K']:.3f}), K-pass bytes {st['kpass_bytes'] / 1e6:.1f} MB, "
          f"32x32 tiles with a kept entry {kept_tiles}/{tiles} ({kept_tiles / tiles:.3f}), "
          f"max rel. error of K^T K b vs the exact solve {err:.3g}", flush=True)
    s.close()
