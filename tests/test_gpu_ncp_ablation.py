"""Min-map NCP (App. B.1) and mass-inverse preconditioner on the GPU vs the
fp64 oracle (the ablation of Fig. 11), through the C ABI
(include/sim.h sim_set_ncp)."""
import math

import numpy as np
import pytest

import scenes
from oracle import oracle as O
import _parity
from _parity import assert_frame_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def simmod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_15078_b200 as m
    return m


@pytest.mark.parametrize("ncp,precond", [(1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("dmu", [+0.05, -0.05])
def test_incline_ncp_variants_resynced(simmod, ncp, precond, dmu):
    """10-degree incline, E = 1e8 (Fig. 11): frames re-synced to the GPU state.  Min-map +
    Delassus: whole frames of 5 L-G iterations, each iteration within 1e-5 bbox of the oracle's
    iteration from the GPU's iterate and the frame within 1e-5 bbox (3x on frames the oracle
    itself shows ill-conditioned: frame 5 of the sliding min-map run moves the fp64 oracle by 0.15
    of the tolerance under fp32 input rounding alone; tests/_parity.py).  With the mass-inverse r
    (h^2/m: orders above h^2 D_jj for a stiff block) the FB / min-map fixed point is not reached in
    5 iterations, so those variants are gated one L-G iteration per frame (10 in a row, plain
    bound) -- the same kernels, one nonlinear step at a time."""
    th = 10.0
    sc = scenes.incline_block(theta_deg=th, mu=math.tan(math.radians(th)) + dmu, nv=5, edge=0.1, youngs=1e8)
    s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    s.set_ncp(ncp, precond)
    s.set_contacts(sc.contacts)
    iters, frames = (5, 6) if precond == 0 else (1, 10)
    o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=iters, ncp=ncp, precond=precond)
    o.set_contacts(sc.contacts)
    tol = 1e-5 * sc.mesh.bbox_diag()
    x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
    for f in range(frames):
        if iters > 1:
            its = _parity.gpu_iterates(s, x, v, iters)
            _parity.assert_iteration_parity(o, x, v, None, its, tol)
        s.set_state(x, v)
        s.step(1, iters)
        xg, vg = s.get_state()
        xo, vo, info = o.frame(x, v)
        if iters > 1:
            _parity.assert_frame_parity_conditioned(o, x, v, xg, xo, tol, what=f"frame {f}")
        else:
            assert_frame_parity(o, x, v, xg, xo, tol, what=f"frame {f}")
        x, v = xg, vg


def test_minmap_small_pile(simmod):
    """Min-map on the 9-cube pile (soft-soft rows), both CR implementations."""
    sc = scenes.pile(cells=3, nx=2, layers=2)
    o = O.Oracle(sc.mesh, sc.material, sc.h, ncp=1)
    o.set_contacts(sc.contacts)
    tol = 1e-5 * sc.mesh.bbox_diag()
    for mode in (1, 2):
        s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
        s.set_cr_mode(mode)
        s.set_ncp(1, 0)
        s.set_contacts(sc.contacts)
        x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
        for f in range(4):
            s.set_state(x, v)
            s.step(1, 5)
            xg, vg = s.get_state()
            xo, _, _ = o.frame(x, v)
            assert np.abs(xg - xo).max() < tol, (mode, f, np.abs(xg - xo).max())
            x, v = xg, vg


def test_preconditioner_values(simmod):
    """r from D_jj vs from [J M^-1 J^T]_jj: the GPU's contact state C diagonal reflects the
    chosen r (min-map inactive-normal rows have E_n = r_n)."""
    from paper_2503_15078_b200._lib import debug_contact_state
    sc = scenes.incline_block(theta_deg=0.0, mu=0.5, nv=4, edge=0.1, youngs=1e6)
    s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    lifted = [scenes.Contact(c.verts, c.weights, c.normal, c.offset - 0.01, mu=c.mu) for c in sc.contacts]
    s.set_contacts(lifted)      # obstacle 1 cm below: every normal row inactive (y > r lam = 0)
    for precond in (0, 1):
        s.set_ncp(1, precond)
        s.step(1, 1)
        st = debug_contact_state(s)
        o = O.Oracle(sc.mesh, sc.material, sc.h, ncp=1, precond=precond)
        o.set_contacts(lifted)
        rn = o.r_row[0::3]
        assert np.allclose(st["cdiag"][0::3] * sc.h ** 2, rn, rtol=1e-6), precond
