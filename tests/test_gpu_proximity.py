"""GPU proximity query (include/sim.h sim_detect_contacts; "simple proximity queries",
PAPER.md L1059-1064) against a numpy reference written here from the
definitions (signed distance to a plane / sphere / capsule surface, nearest obstacle wins,
reading A31), and closed-loop frames that detect their contacts every frame."""
import math

import numpy as np
import pytest

import scenes
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def simmod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_15078_b200 as m
    return m


def reference_query(x, cand, obstacles, margin):
    """(vertex, normal, offset, obstacle) of every candidate within margin, candidate order."""
    out = []
    for v in cand:
        p = x[v]
        best = None
        for k, o in enumerate(obstacles):
            a, b, r = np.asarray(o["a"], float), np.asarray(o.get("b", np.zeros(3)), float), o.get("radius", 0.0)
            if o["kind"] == 0:
                g = float((p - a) @ b)
                n, q = b, p - g * b
            else:
                core = a
                if o["kind"] == 2:
                    d = b - a
                    t = min(max(float((p - a) @ d) / float(d @ d), 0.0), 1.0)
                    core = a + t * d
                w = p - core
                dist = float(np.linalg.norm(w))
                n = w / dist
                g = dist - r
                q = core + r * n
            if g < margin and (best is None or g < best[0]):
                best = (g, n, float(n @ q), k)
        if best is not None:
            out.append((int(v), best[1], best[2], best[3]))
    return out


def test_capsule_query_matches_reference_cfg3(simmod):
    """cfg3's six capsule bars, all free bottom-face vertices as candidates, margin 1 mm."""
    sc = scenes.make_scene("cfg3")
    s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    cand = np.nonzero(sc.mesh.X[:, 2] < 1e-12)[0]
    margin = 1e-3
    n = s.detect_contacts(sc.obstacles, cand, margin)
    ref = reference_query(sc.mesh.X, cand[sc.mesh.fixed[cand] == 0], sc.obstacles, margin)
    assert n == len(ref) > 100
    got = s.get_contacts()
    assert np.array_equal(got["verts"][:, 0], [r[0] for r in ref])
    assert np.abs(got["normal"] - np.array([r[1] for r in ref])).max() < 1e-12
    assert np.abs(got["offset"] - np.array([r[2] for r in ref])).max() < 1e-12
    # the scene's own 800-contact fixture was drawn from the same query: every fixture vertex
    # whose gap is below the margin is detected with the same normal and offset
    fx = {c.verts[0]: c for c in sc.contacts}
    for k, v in enumerate(got["verts"][:, 0]):
        if int(v) in fx:
            assert np.abs(got["normal"][k] - fx[int(v)].normal).max() < 1e-12
            assert abs(got["offset"][k] - fx[int(v)].offset) < 1e-12


def test_mixed_obstacles_moved_state(simmod):
    """Plane + sphere + capsule, deformed state, margin 5 mm: same contact set as the reference."""
    sc = scenes.make_scene("block", nv=6, pinned=False)
    X = sc.mesh.X
    s = simmod.Sim(X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    x, v = scenes.random_state(sc.mesh, seed=12, amp=0.2)
    s.set_state(x, v)
    obst = [{"kind": 0, "a": (0, 0, -0.002), "b": (0, 0, 1.0), "mu": 0.3},
            {"kind": 1, "a": (0.05, 0.05, 0.11), "radius": 0.012, "mu": 0.2},
            {"kind": 2, "a": (-0.01, 0.03, -0.004), "b": (0.11, 0.07, -0.004), "radius": 0.003, "mu": 0.5}]
    cand = np.arange(sc.mesh.n_v)
    n = s.detect_contacts(obst, cand, 5e-3)
    ref = reference_query(x, cand, obst, 5e-3)
    got = s.get_contacts()
    assert n == len(ref) > 10
    assert np.array_equal(got["verts"][:, 0], [r[0] for r in ref])
    assert np.abs(got["normal"] - np.array([r[1] for r in ref])).max() < 1e-12
    assert np.abs(got["offset"] - np.array([r[2] for r in ref])).max() < 1e-12
    assert np.allclose(got["mu"], [obst[r[3]]["mu"] for r in ref])


def test_closed_loop_incline(simmod):
    """cfg2-like incline: contacts detected on the GPU from the plane every frame reproduce the
    fixed bottom-face contact set, and the frames match the oracle fed with the detected set."""
    th = 10.0
    sc = scenes.incline_block(theta_deg=th, mu=math.tan(math.radians(th)) - 0.05, nv=5, edge=0.1, youngs=1e8)
    s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    tol = 1e-5 * sc.mesh.bbox_diag()
    cand = np.arange(sc.mesh.n_v)
    x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
    for f in range(5):
        s.set_state(x, v)
        n = s.detect_contacts(sc.obstacles, cand, 1e-4)
        got = s.get_contacts()
        cs = [scenes.Contact([int(r["verts"][0])], [1.0], r["normal"].copy(), float(r["offset"]),
                             mu=float(r["mu"])) for r in got]
        if f == 0:
            assert n == len(sc.contacts)
        s.step(1, 5)
        xg, vg = s.get_state()
        o.set_contacts(cs)
        xo, _, _ = o.frame(x, v)
        assert np.abs(xg - xo).max() < tol, (f, np.abs(xg - xo).max())
        x, v = xg, vg


def test_schur_reuse_is_bitwise_recompute(simmod):
    """Delassus reuse across commits (include/sim.h sim_set_schur_reuse): a
    block dropping onto a capsule detects its contacts every frame (the set grows and shifts);
    the handle that copies the Gram entries of known vertex pairs and computes only new rows
    produces the same G (bitwise) and the same frames (bitwise) as the one recomputing."""
    sc = scenes.make_scene("block", nv=7, pinned=False)
    X = sc.mesh.X
    obst = [{"kind": 2, "a": (-0.02, 0.06, -0.006), "b": (0.14, 0.05, -0.004), "radius": 0.005, "mu": 0.4},
            {"kind": 0, "a": (0, 0, -0.03), "b": (0, 0, 1.0), "mu": 0.4}]
    cand = np.arange(sc.mesh.n_v)
    hs = []
    for reuse in (False, True):
        s = simmod.Sim(X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
        s.set_schur_reuse(reuse)
        hs.append(s)
    reused_any = False
    for f in range(12):
        counts = [s.detect_contacts(obst, cand, 4e-3) for s in hs]
        assert counts[0] == counts[1]
        if counts[0]:
            cv0, G0 = hs[0].debug_delassus()
            cv1, G1 = hs[1].debug_delassus()
            assert np.array_equal(cv0, cv1) and np.array_equal(G0, G1), f
            st = hs[1].stats()
            reused_any |= st["gram_rows_reused"] > 0 and st["gram_rows_computed"] < st["n_contact_vertices"]
        for s in hs:
            s.step(1, 5)
        x0, v0 = hs[0].get_state()
        x1, v1 = hs[1].get_state()
        assert np.array_equal(x0, x1) and np.array_equal(v0, v1), f
    assert reused_any


def test_schur_reuse_two_commits_between_steps(simmod):
    """Gram reuse while a commit is pending (the second sim_set_contacts before a step on a
    single-scene handle, whose commit's host half runs eagerly): the reused Delassus rows must
    still equal a recomputation bitwise."""
    sc = scenes.incline_block(theta_deg=10.0, mu=0.5, nv=5, edge=0.1, youngs=1e8)
    cs = sc.contacts
    a, b = cs[: len(cs) // 2 + 3], cs[len(cs) // 2 - 3:]
    hs = []
    for reuse in (False, True):
        s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)
        s.set_schur_reuse(reuse)
        s.set_contacts(a)
        s.step(1, 5)
        s.set_contacts(b)          # commit host half (pending device half)
        s.set_contacts(cs)         # second commit before the step
        hs.append(s)
    cv0, G0 = hs[0].debug_delassus()
    cv1, G1 = hs[1].debug_delassus()
    assert np.array_equal(cv0, cv1) and np.array_equal(G0, G1)
    for s in hs:
        s.step(2, 5)
    assert np.array_equal(hs[0].get_state()[0], hs[1].get_state()[0])
