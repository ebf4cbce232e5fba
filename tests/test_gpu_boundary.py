"""The C ABI's state, pin, statistics and allocator calls (include/sim.h), on the GPU."""
import math

import numpy as np
import pytest

import scenes
from oracle import oracle as O
import _parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def simmod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_15078_b200 as m
    return m


def test_set_pins_scripted_handle(simmod):
    """sim_set_pins (moving positional constraint, P:L230 / P:L1241; reading A7): the cantilever's
    fixed end follows a scripted circular path; every frame ends with the pinned vertices on
    their targets and the free vertices matching the oracle given the same Dirichlet targets.
    A frame without a new call continues at the last target velocity."""
    sc = scenes.make_scene("cfg1")
    s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    pinned = np.flatnonzero(sc.mesh.fixed)          # ascending original ids (the call's order)
    assert np.array_equal(pinned, o.pinned)
    x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
    tol = 1e-5 * sc.mesh.bbox_diag()
    for f in range(12):
        ang = 0.4 * (f + 1)
        tgt = sc.mesh.X[pinned] + 0.02 * np.array([math.cos(ang) - 1.0, math.sin(ang), 0.0])
        s.set_pins(tgt)
        s.step(1, 5)
        x, v, _ = o.frame(x, v, pin_targets=tgt)
        xg, vg = s.get_state()
        assert np.abs(xg[pinned] - tgt).max() < 1e-12
        assert np.abs(xg - x).max() <= tol, (f, np.abs(xg - x).max() / tol)
    vp = vg[pinned]                     # the pins' current velocity
    s.step(1, 5)
    x2, _ = s.get_state()
    assert np.abs(x2[pinned] - (tgt + sc.h * vp)).max() < 1e-12
    with pytest.raises(simmod.SimError, match="pinned"):
        s.set_pins(tgt[:-1])


def test_set_pins_per_instance(simmod):
    """Targets are per instance: two instances sharing K, only instance 1's handle moves."""
    sc = scenes.make_scene("cfg1")
    s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=2)
    pinned = np.flatnonzero(sc.mesh.fixed)
    tgt = sc.mesh.X[pinned] + np.array([0.0, 0.01, 0.0])
    s.set_pins(tgt, instance=1)
    s.step(1, 5)
    assert np.abs(s.get_state(0)[0][pinned] - sc.mesh.X[pinned]).max() == 0
    assert np.abs(s.get_state(1)[0][pinned] - tgt).max() < 1e-12


def test_stats_per_instance(simmod):
    """sim_get_stats per instance: contact counts, the frame-end classification (reading A21,
    the oracle's rule on the GPU's x and lambda), cone violation and penetration; instance -1
    sums / maximises over the instances."""
    th = 10.0
    mus = math.tan(math.radians(th))
    scs = [scenes.incline_block(theta_deg=th, mu=mus + d, nv=5, edge=0.1, youngs=1e8) for d in (0.05, -0.05)]
    base = scs[0]
    S = 3
    s = simmod.Sim(base.mesh.X, base.mesh.T, base.mesh.fixed, base.material, base.h, n_instances=S)
    sets = [scs[0].contacts, scs[1].contacts, []]
    s.set_contacts_batch(sets)
    s.step(4, 5)
    total = s.stats(-1)
    per = [s.stats(i) for i in range(S)]
    for i in range(S):
        st = per[i]
        assert st["instance"] == i and st["n_contacts"] == len(sets[i])
        if not sets[i]:
            assert st["n_active"] == st["n_stick"] == st["n_slip"] == 0
            continue
        o = O.Oracle(base.mesh, base.material, base.h)
        o.set_contacts(sets[i])
        x, v = s.get_state(i)
        cls = o.classify(x, x - base.h * v, s.get_lambda(i))
        assert st["n_active"] == int(np.count_nonzero(cls > 0))
        assert st["n_stick"] == int(np.count_nonzero(cls == 1))
        assert st["n_slip"] == int(np.count_nonzero(cls == 2))
        lam = s.get_lambda(i).reshape(-1, 3)
        cone = np.maximum(0, np.linalg.norm(lam[:, 1:], axis=1) - sets[i][0].mu * np.maximum(lam[:, 0], 0))
        assert abs(st["max_cone_violation"] - cone.max()) <= 1e-12 * max(1.0, cone.max())
        pen = np.maximum(0, -(o.Jx(x)[0::3] - o.d_row[0::3])).max()
        assert abs(st["max_penetration"] - pen) <= 1e-12
    assert per[0]["n_active"] > 0 and per[1]["n_active"] > 0 and per[1]["n_slip"] > 0
    for k in ("n_contacts", "n_active", "n_stick", "n_slip", "n_contact_vertices"):
        assert total[k] == sum(p[k] for p in per), k
    assert total["max_cone_violation"] == max(p["max_cone_violation"] for p in per)
    assert total["last_cr_residual"] == max(p["last_cr_residual"] for p in per[:2])
    with pytest.raises(simmod.SimError):
        s.stats(S)


def test_torch_allocator(simmod):
    """sim_set_allocator with PyTorch's caching allocator: the handle's device buffers come from
    torch (torch.cuda.memory_allocated grows by the footprint and drops back on close), and the
    frames are bitwise those of a cudaMalloc handle."""
    import torch
    sc = scenes.make_scene("cfg3")
    ref = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    ref.set_contacts(sc.contacts)
    ref.step(2, 5)
    xr = ref.get_state()[0]
    ref.close()
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_allocated()
    simmod.use_torch_allocator(True)
    try:
        s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
        s.set_contacts(sc.contacts)
        s.step(2, 5)
        xt = s.get_state()[0]
        m1 = torch.cuda.memory_allocated()
        assert m1 - m0 > 2 * 67e6           # K twice (row- and column-major) at least
        s.close()
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated() == m0
    finally:
        simmod.use_torch_allocator(False)
    assert np.array_equal(xt, xr)
