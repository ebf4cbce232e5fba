"""Pins of the fp64 oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it checks (P:L = PAPER.md line, S:L = SPEC.md line)
and is chosen so that a plausible mistake (dropped term, wrong sign or index,
transposed operand) fails it.  No expected value comes from the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.optimize as so

import scenes
from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def rot(axis, ang):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * K @ K


def random_rotations(n, rng):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1)], 1)


# ----------------------------------------------------------------- golden
def test_golden_fb_values():
    for e in GOLD["fb_phi"]:
        phi, _, _ = O.fb_normal(e["y"], e["lam"], e["r"])
        assert abs(float(phi) - e["phi"]) < 1e-14, e["cite"]
    for e in GOLD["fb_theta_n"]:
        _, th, _ = O.fb_normal(e["y"], e["lam"], e["r"])
        assert abs(float(th) - e["theta"]) < 1e-14, e["cite"]


def test_golden_arap():
    for e in GOLD["arap"]:
        P = O.project(np.asarray(e["F"], float)[None], O.ARAP, 1.0, 1.0, 1.0)[0]
        assert np.allclose(P, e["R"], atol=1e-14), e["cite"]


def test_golden_cr_diag():
    for e in GOLD["cr_diag"]:
        A = np.diag(e["A"])
        z, res = O.cr_solve(lambda v: A @ v, np.asarray(e["b"], float), e["iters"])
        assert np.allclose(z, e["x"], atol=1e-14) and res < 1e-14, e["cite"]


def test_golden_preconditioner_and_delassus_closed_form():
    """A -> M when the elastic weight vanishes, so D_jj = 1/M_a exactly
    (P:L858); r_n = h^2 D_jj, r_f = h D_jj.  Density chosen so
    M_1 = 0.25 kg -> D_jj = 4 (S:L350 worked example)."""
    e = GOLD["preconditioner"][0]
    mesh = scenes.single_tet()
    vol = 0.1 ** 3 / 6.0
    rho = 0.25 * 4.0 / vol
    mat = scenes.Material(model=O.ARAP, density=rho, youngs=1e-12, poisson=0.3)
    o = O.Oracle(mesh, mat, e["h"])
    n = np.array([0.0, 0.0, 1.0])
    t1, t2 = scenes.tangent_frame(n)
    o.set_contacts([scenes.Contact([1], [1.0], n, 0.0, mu=0.5, tangent1=t1, tangent2=t2)])
    assert np.allclose(np.diag(o.D), e["Djj"], rtol=1e-9)
    assert abs(o.r_row[0] - e["r_n"]) < 1e-12 and np.allclose(o.r_row[1:], e["r_f"], rtol=1e-9), e["cite"]
    # off-diagonal of one contact's 3 rows: c_j . c_k = 0 for an orthonormal frame
    assert np.allclose(o.D - np.diag(np.diag(o.D)), 0.0, atol=1e-9)


# ------------------------------------------------------------ kinematics
def test_deformation_gradient_special_cases():
    mesh = scenes.cantilever()
    _, _, Bm = None, None, None
    Bm, vol, w, M = O.rest_data(mesh.X, mesh.T, 1000.0, 1.0)
    T = mesh.T.astype(np.int64)
    F = O.deformation_gradients(mesh.X, T, Bm)
    assert np.allclose(F, np.eye(3), atol=1e-12)                      # rest -> I
    R = rot([1, 2, 3], 0.7)
    F = O.deformation_gradients(mesh.X @ R.T + [1, -2, 3], T, Bm)
    assert np.allclose(F, R, atol=1e-12)                              # rigid -> R
    F = O.deformation_gradients(2.0 * mesh.X, T, Bm)
    assert np.allclose(F, 2 * np.eye(3), atol=1e-12)                 # 2x scale
    assert np.all(vol > 0) and abs(vol.sum() - 0.1 * 0.1 * 0.4) < 1e-15
    assert abs(M.sum() - 1000.0 * 0.004) < 1e-12                     # lumped mass = rho V (A6)


def test_system_matrix_kron_structure_and_translation_invariance():
    """A = M + h^2 sum w G^T G assembled explicitly with 9x12 G_i
    (columns from the linear map x -> F) equals A_v (x) I_3; A_v 1 = M."""
    sc = scenes.make_scene("block", nv=3, pinned=False)
    mesh, h = sc.mesh, 0.01
    T = mesh.T.astype(np.int64)
    Bm, vol, w, M = O.rest_data(mesh.X, T, 1000.0, 3.0e5)
    Av = O.assemble_Av(mesh.n_v, T, Bm, w, M, h).toarray()
    n = mesh.n_v
    A3 = np.diag(np.repeat(M, 3))
    for t in range(T.shape[0]):
        G = np.zeros((9, 3 * n))
        for q in range(3 * n):
            e = np.zeros(3 * n)
            e[q] = 1.0
            G[:, q] = O.deformation_gradients(e.reshape(n, 3), T[t:t + 1], Bm[t:t + 1])[0].reshape(-1)
        A3 += h * h * w[t] * G.T @ G
    assert np.allclose(A3, np.kron(Av, np.eye(3)), rtol=0, atol=1e-12 * np.abs(A3).max())
    assert np.allclose(Av @ np.ones(n), M, rtol=1e-12)


def test_global_solve_matches_dense_lu():
    """x = A^-1 b: SuperLU on A_ff vs dense LU (numpy) on cfg1."""
    sc = scenes.make_scene("cfg1")
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    rng = np.random.default_rng(0)
    b = rng.standard_normal((o.free.size, 3))
    x = o.solve(b)
    xd = np.linalg.solve(o.A_ff.toarray(), b)
    assert np.max(np.abs(x - xd)) <= 1e-12 * np.max(np.abs(xd))


# --------------------------------------------------------------- local step
def test_signed_svd():
    rng = np.random.default_rng(1)
    F = rng.standard_normal((200, 3, 3))
    F[::3] = -F[::3]
    U, s, V = O.signed_svd(F)
    assert np.allclose(np.einsum("tij,tj,tkj->tik", U, s, V), F, atol=1e-12)
    assert np.allclose(np.linalg.det(U), 1) and np.allclose(np.linalg.det(V), 1)
    assert np.all(s[:, 0] >= s[:, 1]) and np.all(s[:, 1] >= np.abs(s[:, 2]))
    assert np.all(np.sign(s[:, 2]) == np.sign(np.linalg.det(F)))


def _matrix_objective(model, k, mu, lam, F):
    """Eq. PD local written on the 3x3 matrix P (not in sigma space)."""
    def f(pv):
        P = pv.reshape(3, 3)
        val = 0.5 * k * np.sum((P - F) ** 2)
        if model == O.NEOHOOKEAN:
            J = np.linalg.det(P)
            if J <= 0:
                return 1e30
            val += 0.5 * mu * (np.sum(P * P) - 3) - mu * math.log(J) + 0.5 * lam * math.log(J) ** 2
        else:   # linear corotated (A2): mu|P - R(P)|^2 + lam/2 tr^2(R^T P - I)
            U, s, Vt = np.linalg.svd(P)
            Rp = U @ Vt
            if np.linalg.det(Rp) < 0:
                U[:, 2] *= -1
                Rp = U @ Vt
            val += mu * np.sum((P - Rp) ** 2) + 0.5 * lam * np.trace(Rp.T @ P - np.eye(3)) ** 2
        return val
    return f


@pytest.mark.parametrize("model", [O.NEOHOOKEAN, O.COROTATED])
def test_projection_matches_matrix_space_brute_force(model):
    """sigma-space solution (A2-A5) == direct 9-D minimisation of eq. PD local."""
    mu, lam = O.lame(1e6, 0.3)
    k = 2 * mu
    rng = np.random.default_rng(2 + model)
    for _ in range(6):
        F = rot(rng.standard_normal(3), rng.uniform(0, 3)) @ np.diag(rng.uniform(0.6, 1.5, 3)) @ \
            rot(rng.standard_normal(3), rng.uniform(0, 3))
        P = O.project(F[None], model, k, mu, lam)[0]
        f = _matrix_objective(model, k / mu, 1.0, lam / mu, F)       # scaled by 1/mu
        res = so.minimize(f, P.reshape(-1) + 1e-3 * rng.standard_normal(9), method="BFGS",
                          options={"gtol": 1e-10, "maxiter": 2000})
        assert f(P.reshape(-1)) <= res.fun + 1e-9
        assert np.allclose(res.x.reshape(3, 3), P, atol=2e-5)


@pytest.mark.parametrize("model", [O.NEOHOOKEAN, O.COROTATED, O.ARAP])
def test_projection_rest_and_rotation(model):
    mu, lam = O.lame(1e6, 0.3)
    R = rot([0.3, -1, 2], 1.1)
    P = O.project(np.stack([np.eye(3), R]), model, 2 * mu, mu, lam)
    assert np.allclose(P[0], np.eye(3), atol=1e-12) and np.allclose(P[1], R, atol=1e-12)


def test_nh_kkt_and_inverted():
    """NH minimiser: gradient of eq. PD local vanishes (finite differences of the
    matrix objective); inverted F still gives det p > 0."""
    mu, lam = O.lame(1e6, 0.3)
    k = 2 * mu
    rng = np.random.default_rng(5)
    F = rng.standard_normal((20, 3, 3)) * 0.3 + np.eye(3)
    F[:5] = F[:5] @ np.diag([1, 1, -1])
    P = O.project(F, O.NEOHOOKEAN, k, mu, lam)
    assert np.all(np.linalg.det(P) > 0)
    for t in range(5, 20):
        f = _matrix_objective(O.NEOHOOKEAN, k / mu, 1.0, lam / mu, F[t])
        g = so.approx_fprime(P[t].reshape(-1), f, 1e-7)
        assert np.linalg.norm(g) < 1e-4 * max(1.0, np.linalg.norm(F[t]))


def test_arap_optimal_against_random_rotations():
    rng = np.random.default_rng(3)
    F = rng.standard_normal((3, 3))
    if np.linalg.det(F) < 0:
        F[:, 0] *= -1
    R = O.project(F[None], O.ARAP, 1, 1, 1)[0]
    S = random_rotations(1000, rng)
    assert np.allclose(R.T @ R, np.eye(3), atol=1e-12) and abs(np.linalg.det(R) - 1) < 1e-12
    assert np.linalg.norm(F - R) <= np.min(np.linalg.norm(F[None] - S, axis=(1, 2))) + 1e-12


# ---------------------------------------------------------------- frames
@pytest.mark.parametrize("model", [O.NEOHOOKEAN, O.COROTATED, O.ARAP])
def test_rest_state_is_fixed_point(model):
    """Zero elastic force and energy at rest: b = A X so x stays X."""
    sc = scenes.make_scene("cfg1")
    mat = scenes.Material(model=model, gravity=(0.0, 0.0, 0.0))
    o = O.Oracle(sc.mesh, mat, sc.h)
    x, v, _ = o.frame(sc.mesh.X.copy(), np.zeros_like(sc.mesh.X))
    assert np.max(np.abs(x - sc.mesh.X)) < 1e-13 * sc.mesh.bbox_diag() and np.max(np.abs(v)) < 1e-11


@pytest.mark.parametrize("model", [O.NEOHOOKEAN, O.COROTATED])
def test_free_fall_closed_form(model):
    """No pins or contacts: x_n = x_0 + h^2 g n(n+1)/2, v_n = n h g (implicit
    Euler; G annihilates translations, so one L-G iteration is exact)."""
    sc = scenes.make_scene("cfg1")
    mesh = scenes.Mesh(sc.mesh.X, sc.mesh.T, np.zeros(sc.mesh.n_v, np.uint8))
    mat = scenes.Material(model=model)
    o = O.Oracle(mesh, mat, sc.h)
    g = np.asarray(mat.gravity)
    x, v = mesh.X.copy(), np.zeros_like(mesh.X)
    for n in range(1, 11):
        x, v, _ = o.frame(x, v)
        assert np.max(np.abs(x - (mesh.X + sc.h ** 2 * g * n * (n + 1) / 2))) < 1e-12
        assert np.max(np.abs(v - n * sc.h * g)) < 1e-10


def _random_contacts(o, rng, n):
    free = o.free
    verts = rng.choice(free, size=n + 2, replace=False)
    cs = []
    for i in range(n):
        nrm = rng.standard_normal(3)
        nrm /= np.linalg.norm(nrm)
        t1, t2 = scenes.tangent_frame(nrm)
        cs.append(scenes.Contact([int(verts[i])], [1.0], nrm, rng.standard_normal() * 1e-3,
                                 mu=0.4, tangent1=t1, tangent2=t2))
    nrm = np.array([0.0, 0.0, 1.0])
    t1, t2 = scenes.tangent_frame(nrm)
    cs.append(scenes.Contact([int(verts[n]), int(verts[n + 1])], [0.3, 0.7], nrm, 0.0,
                             mu=0.2, tangent1=t1, tangent2=t2))
    cs.append(scenes.Contact([int(verts[n + 1])], [1.0], np.array([1.0, 0, 0]), 0.01,
                             kind=1, compliance=1e-6))
    return cs


def test_delassus_is_J_Ainv_JT():
    """D = J A^-1 J^T against explicit 3n-DoF J and a dense inverse;
    symmetric and PSD."""
    sc = scenes.make_scene("block", nv=3)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    rng = np.random.default_rng(4)
    cs = _random_contacts(o, rng, 5)
    o.set_contacts(cs)
    nf = o.free.size
    pos = {int(v): i for i, v in enumerate(o.free)}
    J = np.zeros((o.m, 3 * nf))
    for j in range(o.m):
        for q in range(4):
            a = o.rows.verts[j, q]
            if a >= 0:
                J[j, 3 * pos[int(a)]:3 * pos[int(a)] + 3] += o.rows.wts[j, q] * o.rows.c[j]
    A3 = np.kron(o.A_ff.toarray(), np.eye(3))
    D = J @ np.linalg.solve(A3, J.T)
    assert np.allclose(o.D, D, rtol=0, atol=1e-12 * np.abs(D).max())
    assert np.allclose(o.D, o.D.T, atol=1e-15)
    assert np.min(np.linalg.eigvalsh(o.D)) > -1e-12 * np.abs(D).max()


def test_fb_normal_derivatives_are_theta_and_E():
    """Splitting identity: d phi_n/d y = theta_n,
    d phi_n/d lam = E_n  (so H_n = theta_n J_n exactly)."""
    rng = np.random.default_rng(6)
    for _ in range(50):
        y, lam, r = rng.standard_normal(), abs(rng.standard_normal()), abs(rng.standard_normal()) + 0.1
        phi, th, E = O.fb_normal(y, lam, r)
        d = 1e-6
        dy = (O.fb_normal(y + d, lam, r)[0] - O.fb_normal(y - d, lam, r)[0]) / (2 * d)
        dl = (O.fb_normal(y, lam + d, r)[0] - O.fb_normal(y, lam - d, r)[0]) / (2 * d)
        assert abs(dy - th) < 1e-6 and abs(dl - E) < 1e-6
    # theta in [0, 2] (reading A15; y < 0, lam = 0 gives 2)
    assert abs(float(O.fb_normal(-1.0, 0.0, 1.0)[1]) - 2.0) < 1e-15
    assert float(O.fb_normal(0.0, 0.0, 1.0)[1]) == 1.0 and float(O.fb_normal(0.0, 0.0, 1.0)[2]) == 0.0


def test_fb_friction_cases():
    """App. B.2 friction: inactive -> theta 0, E 1; stick inside
    the cone (ydot = 0) -> E 0; on the cone boundary -> E = |ydot|/(mu lam_n),
    the Coulomb ratio of eq. coulomb's law 1."""
    th, E = O.fb_friction(np.array([0.3, 0.1]), np.array([0.0, 0.0]), 0.0, 0.5, 0.2)
    assert th == 0.0 and E == 1.0
    th, E = O.fb_friction(np.zeros(2), np.array([0.1, 0.0]), 1.0, 0.5, 0.2)
    assert th == 1.0 and abs(E) < 1e-15
    yd = np.array([0.3, -0.4])
    lf = -0.5 * 2.0 * yd / np.linalg.norm(yd)          # |lam_f| = mu lam_n, opposing
    th, E = O.fb_friction(yd, lf, 2.0, 0.5, 0.07)
    assert abs(E - np.linalg.norm(yd) / (0.5 * 2.0)) < 1e-12
    # the 0/0 point has limit 0 (reading A16)
    th, E = O.fb_friction(np.array([1e-12, 0.0]), np.zeros(2), 1.0, 0.5, 0.2)
    assert 0.0 <= E < 1e-9
    # degenerate cone mu = 0 uses the inactive branch (reading A16b)
    th, E = O.fb_friction(np.array([0.3, 0.0]), np.zeros(2), 1.0, 0.0, 0.2)
    assert th == 0.0 and E == 1.0


def test_fb_friction_outside_cone_branch():
    """Reading A16c: E_f is evaluated at the cone projection of lam_f,
    q = mu lam_n - min(|lam_f|, mu lam_n).  The printed formula is kept inside
    the cone; there its s = 0 value is 0 (stick) and as |lam_f| -> mu lam_n from inside E_f tends
    to |ydot|/(mu lam_n).  On and outside the cone E_f = |ydot|/(mu lam_n) exactly, for every
    |lam_f| -- including |lam_f| > 2 mu lam_n, where the printed q would put the denominator
    phi_FB(s, q) + r |lam_f| through zero (a pole) and below it (anti-dissipative E_f < 0).
    Over a sweep of states E_f is finite, >= 0 and <= |ydot| / min(|lam_f|, mu lam_n)."""
    mu, ln, r = 0.5, 2.0, 0.3
    yd = np.array([0.12, -0.05])
    s = float(np.linalg.norm(yd))
    coulomb = s / (mu * ln)
    for f in (1.0, 1.5, 1.99, 2.0, 2.01, 3.0, 40.0):     # on / outside the cone (the printed pole at f = 2)
        _, E = O.fb_friction(yd, np.array([0.0, f * mu * ln]), ln, mu, r)
        assert abs(E - coulomb) <= 1e-12 * coulomb, (f, E, coulomb)
        _, E0 = O.fb_friction(np.zeros(2), np.array([f * mu * ln, 0.0]), ln, mu, r)
        assert E0 == 0.0                                  # s = 0: no slip, no compliance
    for f in (0.0, 0.3, 0.9):                             # inside: the printed formula, s = 0 -> 0
        _, E0 = O.fb_friction(np.zeros(2), np.array([f * mu * ln, 0.0]), ln, mu, r)
        assert E0 == 0.0
    # continuity across the cone boundary, from inside
    _, Ein = O.fb_friction(yd, np.array([(1 - 1e-9) * mu * ln, 0.0]), ln, mu, r)
    assert abs(Ein - coulomb) < 1e-6 * coulomb
    # inside the cone with s > 0: the printed expression written out
    lf = np.array([0.4, 0.2])
    q = mu * ln - np.linalg.norm(lf)
    R = math.sqrt(s * s + r * r * q * q)
    _, E = O.fb_friction(yd, lf, ln, mu, r)
    assert abs(E - r * (R - r * q) / (s + mu * r * ln - R)) < 1e-12 * E
    rng = np.random.default_rng(11)
    for _ in range(2000):
        ydr = rng.standard_normal(2) * 10.0 ** rng.uniform(-6, 1)
        lfr = rng.standard_normal(2) * 10.0 ** rng.uniform(-3, 1)
        lnr = 10.0 ** rng.uniform(-3, 1)
        _, E = O.fb_friction(ydr, lfr, lnr, 0.5, 10.0 ** rng.uniform(-4, 0))
        bound = np.linalg.norm(ydr) / min(np.linalg.norm(lfr), 0.5 * lnr)
        assert np.isfinite(E) and 0.0 <= E <= bound * (1 + 1e-6), (E, bound)


def _one_contact_oracle(mu=0.5, v_obs=(0.0, 0.0, 0.0)):
    mesh = scenes.single_tet()
    mat = scenes.Material(model=O.NEOHOOKEAN, youngs=1e5)
    o = O.Oracle(mesh, mat, 0.01)
    n = np.array([0.0, 0.0, 1.0])
    t1, t2 = scenes.tangent_frame(n)
    o.set_contacts([scenes.Contact([0], [1.0], n, 0.0, mu=mu, tangent1=t1, tangent2=t2,
                                   obstacle_velocity=np.asarray(v_obs, float))])
    return o, mesh.X, t1, t2


def test_classify_hand_built_states():
    """Frame-end classification (reading A21; P:L292-298 Signorini-Coulomb sets A / I,
    P:L1650 stick/slip case split): inactive iff lambda_n <= 0; stick iff
    |ydot_f| <= r_f (mu lambda_n - |lambda_f|); slip otherwise.  Hand-built (x, x_t, lambda) of
    one vertex contact, ydot_f from x - x_t along t1 (h ydot_f = J_f (x - x_t) - h d_f)."""
    o, X, t1, t2 = _one_contact_oracle()
    h, r = o.h, o.r_row[1]
    lam = np.array([1.0, 0.1, 0.0])               # inside the cone: mu lam_n - |lam_f| = 0.4
    cap = r * 0.4                                 # the stick speed bound
    def state(speed):
        x = X.copy()
        x[0] += h * speed * t1
        return x
    assert O.Oracle.classify(o, X, X, np.array([0.0, 0.0, 0.0]))[0] == 0
    assert O.Oracle.classify(o, X, X, np.array([-1e-3, 0.1, 0.0]))[0] == 0   # lambda_n < 0: inactive
    assert O.Oracle.classify(o, X, X, lam)[0] == 1                            # at rest: stick
    assert O.Oracle.classify(o, state(0.5 * cap), X, lam)[0] == 1
    assert O.Oracle.classify(o, state(2.0 * cap), X, lam)[0] == 2
    # on the cone (|lambda_f| = mu lambda_n) any motion is slip; zero motion is still stick
    on = np.array([1.0, 0.3, 0.4])
    assert O.Oracle.classify(o, X, X, on)[0] == 1
    assert O.Oracle.classify(o, state(1e-9), X, on)[0] == 2
    # outside the cone: slip even at rest
    assert O.Oracle.classify(o, X, X, np.array([1.0, 0.6, 0.0]))[0] == 2


def test_classify_moving_obstacle_relative_velocity():
    """d_f = t . v_obstacle (reading A24): a vertex moving WITH the obstacle has
    zero relative tangential velocity and sticks; a vertex at rest under a moving obstacle
    slides relative to it."""
    vo = np.array([0.2, -0.1, 0.0])
    o, X, t1, t2 = _one_contact_oracle(v_obs=vo)
    lam = np.array([1.0, 0.1, 0.0])
    x = X.copy()
    x[0] += o.h * vo
    assert O.Oracle.classify(o, x, X, lam)[0] == 1
    assert O.Oracle.classify(o, X, X, lam)[0] == 2


def test_carry_multipliers():
    """Reading A10: lambda survives a contact commit for the same constraint (kind, vertices,
    weights, row directions; wherever it sits in the new order), and a changed or new contact
    starts from 0."""
    n = np.array([0.0, 0.0, 1.0])
    t1, t2 = scenes.tangent_frame(n)
    a = scenes.Contact([0], [1.0], n, 0.0, mu=0.5, tangent1=t1, tangent2=t2)
    b = scenes.Contact([1], [1.0], n, 0.0, mu=0.5, tangent1=t1, tangent2=t2)
    c = scenes.Contact([2], [1.0], n, 0.3, mu=0.2, tangent1=t1, tangent2=t2)   # offset / mu may change
    bil = scenes.Contact([3], [1.0], n, 0.0, kind=1, compliance=1e-3)
    old = [a, b, bil]
    lam = np.arange(1.0, 8.0)
    assert np.array_equal(O.carry_multipliers(old, lam, old), lam)
    c2 = scenes.Contact([1], [1.0], n, 0.3, mu=0.2, tangent1=t1, tangent2=t2)
    got = O.carry_multipliers(old, lam, [a, c2, bil])
    assert np.array_equal(got, lam)                                   # same constraint rows
    got = O.carry_multipliers(old, lam, [b, a, bil, c])               # reordered + one more
    assert np.array_equal(got, np.r_[lam[3:6], lam[0:3], 7.0, np.zeros(3)])
    got = O.carry_multipliers(old, lam, [a, a])                       # each old row is used once
    assert np.array_equal(got, np.r_[lam[0:3], np.zeros(3)])
    tilt = scenes.Contact([0], [1.0], n, 0.0, mu=0.5, tangent1=t2, tangent2=-t1)
    assert np.array_equal(O.carry_multipliers(old, lam, [tilt]), np.zeros(3))
    assert np.array_equal(O.carry_multipliers([], None, [a]), np.zeros(3))


def test_cr_equals_dense_solve_after_n_steps():
    """N-step CR on an N x N SPD system is exact (Krylov property)."""
    rng = np.random.default_rng(7)
    for n in (3, 8, 20):
        Q = rng.standard_normal((n, n))
        A = Q @ Q.T + n * np.eye(n)
        b = rng.standard_normal(n)
        z, _ = O.cr_solve(lambda v: A @ v, b, n)
        assert np.allclose(z, np.linalg.solve(A, b), rtol=1e-9, atol=1e-12)
        z0, _ = O.cr_solve(lambda v: A @ v, np.zeros(n), n)
        assert not np.any(z0)


def _floor_tet(mu):
    mesh = scenes.single_tet()
    n = np.array([0.0, 0.0, 1.0])
    t1, t2 = scenes.tangent_frame(n)
    cs = [scenes.Contact([v], [1.0], n, 0.0, mu=mu, tangent1=t1, tangent2=t2) for v in (0, 1, 2)]
    return mesh, cs


def test_contact_statics_force_balance():
    """Resting tet on a floor: converged sum lam_n = m g, the tangential
    forces cancel and stay in the cone, the body stays (Signorini and
    Coulomb)."""
    mesh, cs = _floor_tet(0.5)
    mat = scenes.Material(model=O.NEOHOOKEAN, youngs=1e7)
    o = O.Oracle(mesh, mat, 0.01, lg_iters=40, cr_iters=40)
    o.set_contacts(cs)
    x, v = mesh.X.copy(), np.zeros_like(mesh.X)
    for _ in range(20):
        x, v, info = o.frame(x, v)
    lam = info["lam"].reshape(-1, 3)
    mg = o.M.sum() * 9.81
    assert abs(lam[:, 0].sum() - mg) < 1e-9 * mg
    assert np.all(np.abs(lam[:, 1:].sum(0)) < 1e-9 * mg)
    assert np.all(np.linalg.norm(lam[:, 1:], axis=1) <= 0.5 * lam[:, 0] + 1e-12)
    assert np.max(np.abs(v)) < 1e-9


def test_frictionless_momentum_conservation():
    """mu = 0: lam_f stays 0 and tangential momentum is conserved."""
    mesh, cs = _floor_tet(0.0)
    mat = scenes.Material(model=O.NEOHOOKEAN, youngs=1e5)
    o = O.Oracle(mesh, mat, 0.01, lg_iters=10, cr_iters=10)
    o.set_contacts(cs)
    x = mesh.X.copy()
    v = np.zeros_like(x)
    v[:, 0] = 0.2
    p0 = (o.M[:, None] * v)[:, :2].sum(0)
    for _ in range(5):
        x, v, info = o.frame(x, v)
    lam = info["lam"].reshape(-1, 3)
    assert np.all(lam[:, 1:] == 0.0)
    assert np.allclose((o.M[:, None] * v)[:, :2].sum(0), p0, atol=1e-12)


def _incline_run(dmu, precond, frames=60, nv=4, warm=True):
    """cfg2-type block on the 10-degree slope of Fig. 11 (rho = 1000, E = 1e8),
    10 L-G / 24 CR iterations; mean down-slope velocity after every frame.
    warm: readings A9w/A10w (x^0 = x_t + h v_t, lambda carried across frames)."""
    th = 10.0
    mus = math.tan(math.radians(th))
    sc = scenes.incline_block(theta_deg=th, mu=mus + dmu, nv=nv, edge=0.1, youngs=1e8)
    o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=10, cr_iters=24, precond=precond, warm_start=warm)
    o.set_contacts(sc.contacts)
    x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
    down = -np.array([math.cos(math.radians(th)), 0, math.sin(math.radians(th))])
    lam, vs = None, []
    for _ in range(frames):
        x, v, info = o.frame(x, v, lam0=lam if warm else None)
        lam = info["lam"]
        vs.append(float((v @ down).mean()))
    a = 9.81 * (math.sin(math.radians(th)) - (mus + dmu) * math.cos(math.radians(th)))
    return o, x, np.array(vs), a, sc.h


@pytest.mark.parametrize("dmu,slides", [(+0.001, False), (-0.001, True)])
def test_incline_stick_slip_threshold(dmu, slides):
    """Fig. 11: FB + the Delassus preconditioner resolve the stick/slide switch
    at mu* = tan(10 deg) = 0.17632698 to 0.001.  The down-slope acceleration over frames 70-120
    (after the start transient, which at mu* - 0.001 lasts ~60 frames) is the rigid-limit closed form a = g (sin th - mu cos th)
    within 5 % at mu* - 0.001, and below 5 % of |a| at mu* + 0.001 (stick), in the warm-start
    reading (A9w: x^0 = x_t + h v_t, A10w: lambda carried across frames), the one that reproduces
    the paper's 0.001.  The default reading (x^0 = s, lambda^0 = 0) creeps
    near the threshold: it resolves 0.01 (test_incline_default_reading_resolution)."""
    o, x, vs, a, h = _incline_run(dmu, O.PRECOND_DELASSUS, frames=120)
    acc = (vs[119] - vs[69]) / (50 * h)
    if slides:
        assert abs(acc - a) < 0.05 * a, (acc, a)
    else:
        assert abs(acc) < 0.05 * abs(a), (acc, a)
    # normal penetration stays at rounding level
    assert np.max(-(o.Jx(x)[0::3] - o.d_row[0::3])) < 1e-6


@pytest.mark.parametrize("dmu,slides", [(+0.01, False), (-0.01, True)])
def test_incline_default_reading_resolution(dmu, slides):
    """Default reading (A9: x^0 = s, A10: lambda^0 = 0 every frame), the same Fig. 11 block:
    the switch is resolved at mu* -+ 0.01 (slide acceleration within 5 % of the closed form;
    stick: below 5 % of |a|), one decade coarser than the warm-start reading."""
    o, x, vs, a, h = _incline_run(dmu, O.PRECOND_DELASSUS, warm=False)
    acc = (vs[59] - vs[29]) / (30 * h)
    if slides:
        assert abs(acc - a) < 0.05 * a, (acc, a)
    else:
        assert abs(acc) < 0.05 * abs(a), (acc, a)


def test_incline_mass_inverse_sticks():
    """Fig. 11's ablation: with Macklin's mass-inverse preconditioner
     the block at mu* - 0.01 shows the "undesired sticking behavior" -- its
    acceleration stays below half of the closed form -- while FB + Delassus reaches the closed
    form within 1 %."""
    _, _, vd, a, h = _incline_run(-0.01, O.PRECOND_DELASSUS)
    _, _, vm, _, _ = _incline_run(-0.01, O.PRECOND_MASS)
    acc_d = (vd[59] - vd[29]) / (30 * h)
    acc_m = (vm[59] - vm[29]) / (30 * h)
    assert abs(acc_d - a) < 0.01 * a, (acc_d, a)
    assert acc_m < 0.5 * a, (acc_m, a)


def test_zero_penetration_at_convergence():
    """Elevated budgets: min y_n >= -1e-6 bbox and |phi_FB| small."""
    sc = scenes.incline_block(theta_deg=0.0, mu=0.5, nv=3, edge=0.1, youngs=1e6)
    o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=60, cr_iters=60)
    o.set_contacts(sc.contacts)
    x, v = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
    v[:, 2] = -0.3
    for _ in range(3):
        x, v, info = o.frame(x, v)
    yn = o.Jx(x)[0::3] - o.d_row[0::3]
    assert yn.min() >= -1e-6 * sc.mesh.bbox_diag()
    lam_n = info["lam"][0::3]
    phi, _, _ = O.fb_normal(yn, lam_n, o.r_row[0::3])
    assert np.max(np.abs(phi)) < 1e-6 * max(1.0, o.r_row[0])


# ------------------------------------------- min-map + mass-inverse ablation (NEXT row 1)
def test_golden_minmap_values():
    for e in GOLD["minmap_phi"]:
        phi, _, _ = O.minmap_normal(e["y"], e["lam"], e["r"])
        assert float(phi) == e["phi"], e["cite"]
    for e in GOLD["minmap_normal_case"]:
        _, th, E = O.minmap_normal(e["y"], e["lam"], e["r"])
        assert float(th) == e["theta"] and float(E) == e["E"], e["cite"]


def test_minmap_derivatives_and_complementarity():
    """App. B.1: theta_n = d phi/d y and E_n = d phi/d lam off the kink y = r lam; phi = 0
    exactly on the complementarity set {y = 0 <= lam} U {lam = 0 <= y}."""
    rng = np.random.default_rng(11)
    for _ in range(50):
        y, lam, r = rng.standard_normal(), abs(rng.standard_normal()), abs(rng.standard_normal()) + 0.1
        if abs(y - r * lam) < 1e-3:
            continue
        phi, th, E = O.minmap_normal(y, lam, r)
        d = 1e-7
        dy = (O.minmap_normal(y + d, lam, r)[0] - O.minmap_normal(y - d, lam, r)[0]) / (2 * d)
        dl = (O.minmap_normal(y, lam + d, r)[0] - O.minmap_normal(y, lam - d, r)[0]) / (2 * d)
        assert abs(dy - th) < 1e-6 and abs(dl - E) < 1e-6
    for lam in (0.0, 0.3, 7.0):
        assert float(O.minmap_normal(0.0, lam, 0.5)[0]) == 0.0
    for y in (0.0, 0.2, 3.0):
        assert float(O.minmap_normal(y, 0.0, 0.5)[0]) == 0.0


def test_minmap_friction_cases():
    """App. B.1 friction: inactive -> theta 0, E = I; stick (|ydot| <=
    r(mu lam_n - |lam_f|)) -> E = 0; slip -> E = (|ydot| - r q)/(mu lam_n), which on the
    cone boundary (q = 0) makes phi_f = ydot + |ydot|/(mu lam_n) lam_f vanish exactly for
    the maximal-dissipation force lam_f = -mu lam_n ydot/|ydot|."""
    th, E = O.minmap_friction(np.array([0.3, 0.1]), np.zeros(2), 0.0, 0.5, 0.2)
    assert th == 0.0 and E == 1.0
    th, E = O.minmap_friction(np.array([0.01, 0.0]), np.array([0.1, 0.0]), 1.0, 0.5, 0.2)
    assert th == 1.0 and E == 0.0            # 0.01 <= 0.2 (0.5 - 0.1)
    yd = np.array([0.3, -0.4])
    lf = -0.5 * 2.0 * yd / np.linalg.norm(yd)
    th, E = O.minmap_friction(yd, lf, 2.0, 0.5, 0.07)
    assert abs(E - np.linalg.norm(yd) / (0.5 * 2.0)) < 1e-15
    assert np.abs(th * yd + E * lf).max() < 1e-15
    th, E = O.minmap_friction(np.array([0.3, 0.0]), np.zeros(2), 1.0, 0.0, 0.2)
    assert th == 0.0 and E == 1.0


def test_mass_inverse_preconditioner_closed_form():
    """r_n = h^2 [J M^-1 J^T]_jj, r_f = h [J M^-1 J^T]_jj.  One vertex of mass
    m: 1/m; a soft-soft row x_a - sum b_i x_i: 1/m_a + sum b_i^2/m_i (c unit)."""
    mesh = scenes.single_tet()
    vol = 0.1 ** 3 / 6.0
    mat = scenes.Material(model=O.ARAP, density=1000.0, youngs=1e6, poisson=0.3)
    h = 0.01
    o = O.Oracle(mesh, mat, h, precond=O.PRECOND_MASS)
    m = 1000.0 * vol / 4.0
    n = np.array([0.0, 0.0, 1.0])
    o.set_contacts([scenes.Contact([1], [1.0], n, 0.0, mu=0.5),
                    scenes.Contact([3, 0, 1, 2], [1.0, -0.2, -0.3, -0.5], n, 0.0, mu=0.5)])
    assert abs(o.r_row[0] - h * h / m) < 1e-12 * h * h / m
    assert np.allclose(o.r_row[1:3], h / m, rtol=1e-12)
    q = (1.0 + 0.04 + 0.09 + 0.25) / m
    assert abs(o.r_row[3] - h * h * q) < 1e-12 * h * h * q and np.allclose(o.r_row[4:6], h * q, rtol=1e-12)
    # the Delassus diagonal is larger than the mass-inverse one only through A^-1 <= M^-1 ... (A = M + h^2 L)
    od = O.Oracle(mesh, mat, h)
    od.set_contacts(o.contacts)
    assert np.all(od.r_row <= o.r_row * (1 + 1e-12))


def test_minmap_contact_statics():
    """With min-map (App. B.1) the resting-contact statics of S:L389 hold as with FB:
    converged sum lam_n = m g, tangential forces cancel and stay in the cone, body at rest."""
    mesh, cs = _floor_tet(0.5)
    mat = scenes.Material(model=O.NEOHOOKEAN, youngs=1e7)
    o = O.Oracle(mesh, mat, 0.01, lg_iters=40, cr_iters=40, ncp=O.NCP_MINMAP)
    o.set_contacts(cs)
    x, v = mesh.X.copy(), np.zeros_like(mesh.X)
    for _ in range(20):
        x, v, info = o.frame(x, v)
    lam = info["lam"].reshape(-1, 3)
    mg = o.M.sum() * 9.81
    assert abs(lam[:, 0].sum() - mg) < 1e-9 * mg
    assert np.all(np.abs(lam[:, 1:].sum(0)) < 1e-9 * mg)
    assert np.all(np.linalg.norm(lam[:, 1:], axis=1) <= 0.5 * lam[:, 0] + 1e-12)
    assert np.max(np.abs(v)) < 1e-9


# ------------------------------------------------------------- ADMM-PD (NEXT row 2)
def _psi_nh(F, mu, lam):
    """Compressible Neo-Hookean energy density (reading A3)."""
    J = np.linalg.det(F)
    return 0.5 * mu * (np.sum(F * F) - 3.0) - mu * np.log(J) + 0.5 * lam * np.log(J) ** 2


def _psi_corot(F, mu, lam):
    """Linear corotational energy density (reading A2), R = polar rotation of F."""
    U, _, Vt = np.linalg.svd(F)
    R = U @ Vt
    if np.linalg.det(R) < 0:
        U[:, -1] *= -1
        R = U @ Vt
    return mu * np.sum((F - R) ** 2) + 0.5 * lam * np.trace(R.T @ F - np.eye(3)) ** 2


def _implicit_euler_gradient(o, x, s, psi):
    """h^2 * grad of E(x) = 1/(2h^2) |x - s|_M^2 + sum_i vol_i psi(F_i(x))  (eq. implicit
    euler) at the free vertices; dpsi/dF by central differences, written out
    per tet from Dm and Ds (no oracle helper)."""
    r = o.M[:, None] * (x - s)
    for t in range(o.T.shape[0]):
        v = o.T[t]
        Dm = np.stack([o.X[v[i]] - o.X[v[0]] for i in (1, 2, 3)], 1)
        Bm = np.linalg.inv(Dm)
        F = np.stack([x[v[i]] - x[v[0]] for i in (1, 2, 3)], 1) @ Bm
        vol = abs(np.linalg.det(Dm)) / 6.0
        P = np.zeros((3, 3))
        e = 1e-6
        for i in range(3):
            for j in range(3):
                Fp, Fm = F.copy(), F.copy()
                Fp[i, j] += e
                Fm[i, j] -= e
                P[i, j] = (psi(Fp) - psi(Fm)) / (2 * e)
        g = vol * P @ Bm.T
        for a in range(3):
            r[v[a + 1]] += o.h ** 2 * g[:, a]
        r[v[0]] -= o.h ** 2 * g.sum(1)
    return r[o.free]


@pytest.mark.parametrize("model,psi", [(O.NEOHOOKEAN, _psi_nh), (O.COROTATED, _psi_corot)])
def test_admm_pd_fixed_point_is_implicit_euler(model, psi):
    """ADMM-PD (Overby et al. 2017): at its fixed point z = F and u = grad psi / k,
    so the global step is the stationarity condition M (x - s) + h^2 sum vol G^T dpsi/dF = 0
    of the implicit-Euler objective -- which plain PD without the dual misses (reading A32,
    the Moreau-envelope bias).  Cantilever (cfg1), one frame from rest, 60 L-G iterations."""
    sc = scenes.make_scene("cfg1", model=model)
    res = {}
    for admm in (False, True):
        o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=60, admm=admm)
        x0, v0 = sc.mesh.X.copy(), np.zeros_like(sc.mesh.X)
        s = x0 + sc.h * v0 + sc.h ** 2 * o.g
        x, _, _ = o.frame(x0, v0)
        scale = np.abs(o.M[:, None] * (x - s))[o.free].max()
        res[admm] = np.abs(_implicit_euler_gradient(o, x, s, lambda F: psi(F, o.mu, o.lam))).max() / scale
    assert res[True] < 1e-5, res
    assert res[False] > 100 * res[True], res
