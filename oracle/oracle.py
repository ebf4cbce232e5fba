"""Plain, slow, obviously-correct fp64 oracle of the per-iteration hot path of
arXiv 2503.15078 (Alg. 4) -- TEST INFRASTRUCTURE ONLY.

Citation convention: ``P:L<n>`` = /root/reference/PAPER.md line n (that file
is not read at run time).  Readings of silent/garbled passages are the A-items
of SURVEY.md §8(c), restated in DESIGN.md §3.

What this module computes and how (no blocking, fusion or reordering beyond
the paper's own definitions):

* rest data        Dm, Bm = Dm^-1, vol, lumped M (A6), w_i = k vol_i (A1).
* system           A = M + h^2 sum_i w_i G_i^T G_i  (eq. PD global).
                   Assembled at vertex level A_v; A = A_v (x) I_3 (pinned by a
                   test against the explicit 12x12 per-tet G_i^T G_i assembly).
                   Dirichlet pins by elimination (A7).
* global solve     x = A^-1 b by sparse LU (scipy SuperLU) -- the plain
                   definition; NOT the sparse inverse K (Thm 1 / Alg. 2).
* local step       p_i = argmin w/2|p - F_i|^2 + Psi(p)   (eq. PD local)
                   via numpy's SVD + per-material sigma-space solve (A2-A5).
* contacts         J rows (App. A), D = J A^-1 J^T by direct
                   solves (eq. schur-complement, plain definition),
                   r_n = h^2 D_jj, r_f = h D_jj -- or, for the
                   ablation, the mass-inverse r from [J M^-1 J^T]_jj,
                   FB indicators (App. B.2; readings A14-A16) --
                   or min-map (App. B.1),
                   Schur RHS with the Alg. 3/4 sign (A11),
                   CR (Saad Alg. 6.20) with exactly N_CR iterations (A19),
                   lambda update (no projection, A20) + corrected global solve.
* frame            default (A9, A10): x^0 = s, lambda^0 = 0 every frame;
                   warm_start=True (A9w, A10w): x^0 = x_t + h v_t and lambda^0 = the previous
                   frame's lambda (Alg. 4 never resets it), carried across contact sets by
                   carry_multipliers -- the reading that reproduces Fig. 11's 0.001.

Parity pinning status (see tests/test_oracle_*.py): every function below is
pinned by a closed form, an invariant, a library special case or brute force,
EXCEPT the multi-iteration contact trajectory at real-time budgets and the NH
cantilever deflection, which have no closed form ("parity unpinned" there;
they are compared GPU-vs-oracle only).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "lame", "rest_data", "assemble_Av", "deformation_gradients", "signed_svd",
    "project_sigma", "project", "elastic_forces", "Oracle", "cr_solve",
    "fb_normal", "fb_friction", "minmap_normal", "minmap_friction", "contact_rows", "carry_multipliers",
]

NCP_FB, NCP_MINMAP = 0, 1                  # NCP function (App. B)
PRECOND_DELASSUS, PRECOND_MASS = 0, 1      # complementarity preconditioner (P:L873-880 / P:L918-925)

NEOHOOKEAN, COROTATED, ARAP = 0, 1, 2


# ---------------------------------------------------------------------------
# rest data
# ---------------------------------------------------------------------------
def lame(E: float, nu: float):
    """Lame parameters from (E, nu) (Table 3 columns)."""
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return mu, lam


def rest_data(X: np.ndarray, T: np.ndarray, density: float, k_proj: float):
    """Per-tet Dm^-1, volume, w_i = k vol_i (A1) and lumped mass (A6)."""
    x0 = X[T[:, 0]]
    Dm = np.stack([X[T[:, 1]] - x0, X[T[:, 2]] - x0, X[T[:, 3]] - x0], axis=2)  # columns
    det = np.linalg.det(Dm)
    if np.any(np.abs(det) <= 0.0):
        bad = int(np.nonzero(np.abs(det) <= 0.0)[0][0])
        raise ValueError(f"degenerate tet {bad}")
    Bm = np.linalg.inv(Dm)
    vol = np.abs(det) / 6.0
    w = k_proj * vol
    M = np.zeros(X.shape[0])
    np.add.at(M, T.reshape(-1), np.repeat(density * vol / 4.0, 4))
    return Bm, vol, w, M


def shape_gradients(Bm: np.ndarray):
    """g_a for a = 0..3 with F = sum_a x_a g_a^T: g_a = row a-1 of Bm
    (a = 1..3), g_0 = -sum.  Returns [n_t, 4, 3]."""
    g = np.empty((Bm.shape[0], 4, 3))
    g[:, 1:, :] = Bm
    g[:, 0, :] = -Bm.sum(axis=1)
    return g


def assemble_Av(n_v: int, T: np.ndarray, Bm: np.ndarray, w: np.ndarray, M: np.ndarray, h: float):
    """Vertex-level A_v = M + h^2 sum_i w_i (g_a . g_b)  (eq. PD global P:L321)."""
    g = shape_gradients(Bm)
    gg = np.einsum("tad,tbd->tab", g, g) * (h * h * w)[:, None, None]
    rows = np.repeat(T[:, :, None], 4, axis=2).reshape(-1)
    cols = np.repeat(T[:, None, :], 4, axis=1).reshape(-1)
    A = sp.coo_matrix((gg.reshape(-1), (rows, cols)), shape=(n_v, n_v)).tocsr()
    A = A + sp.diags(M)
    return A.tocsr()


# ---------------------------------------------------------------------------
# local step
# ---------------------------------------------------------------------------
def deformation_gradients(x: np.ndarray, T: np.ndarray, Bm: np.ndarray):
    """F_i = Ds(x) Dm^-1 (G_i x of eq. PD local)."""
    x0 = x[T[:, 0]]
    Ds = np.stack([x[T[:, 1]] - x0, x[T[:, 2]] - x0, x[T[:, 3]] - x0], axis=2)
    return Ds @ Bm


def signed_svd(F: np.ndarray):
    """Signed SVD (reading A5): U, V in SO(3), s1 >= s2 >= |s3|, s3 < 0 iff det F < 0."""
    U, s, Vt = np.linalg.svd(F)
    V = np.swapaxes(Vt, -1, -2).copy()
    U = U.copy()
    s = s.copy()
    du = np.linalg.det(U) < 0
    U[du, :, 2] *= -1.0
    s[du, 2] *= -1.0
    dv = np.linalg.det(V) < 0
    V[dv, :, 2] *= -1.0
    s[dv, 2] *= -1.0
    return U, s, V


def _nh_f(p, sig, k, mu, lam):
    J = np.prod(p, axis=1)
    lnJ = np.log(J)
    return (0.5 * k * ((p - sig) ** 2).sum(1) + 0.5 * mu * ((p * p).sum(1) - 3.0)
            - mu * lnJ + 0.5 * lam * lnJ * lnJ)


def _nh_grad_hess(p, sig, k, mu, lam):
    lnJ = np.log(np.prod(p, axis=1))
    inv = 1.0 / p
    grad = k * (p - sig) + mu * p - mu * inv + lam * lnJ[:, None] * inv
    H = lam * inv[:, :, None] * inv[:, None, :]
    d = k + mu + (mu - lam * lnJ)[:, None] * inv * inv
    H[:, [0, 1, 2], [0, 1, 2]] += d
    return grad, H


def project_sigma(sig: np.ndarray, model: int, k: float, mu: float, lam: float,
                  tol: float = 1e-12, max_iter: int = 200):
    """p* = argmin_p k/2 |p - sigma|^2 + psi(p) in signed-singular-value space.

    ARAP: psi = indicator of SO(3) -> p* = (1, 1, 1).
    Linear corotated (A2, "linear co-rotational" P:L1165): psi = mu sum(p-1)^2 +
      lam/2 (sum p - 3)^2 -> closed form S = (k sum sig + 6mu + 9lam)/(k + 2mu + 3lam),
      p_i = (k sig_i + 2mu - lam (S - 3))/(k + 2mu).
    Neo-Hookean (A3): psi = mu/2 (sum p^2 - 3) - mu ln J + lam/2 ln^2 J, J = prod p;
      damped Newton (A4) from p0 = max(sig, 0.05), backtracking keeps p > 0,
      until |grad| <= tol*k*max(1,|sig|).
    """
    sig = np.asarray(sig, dtype=np.float64)
    if model == ARAP:
        return np.ones_like(sig)
    if model == COROTATED:
        S = (k * sig.sum(1) + 6 * mu + 9 * lam) / (k + 2 * mu + 3 * lam)
        return (k * sig + 2 * mu - lam * (S - 3.0)[:, None]) / (k + 2 * mu)
    if model != NEOHOOKEAN:
        raise ValueError(model)
    p = np.maximum(sig, 0.05)
    scale = np.maximum(1.0, np.linalg.norm(sig, axis=1))
    active = np.ones(sig.shape[0], dtype=bool)
    for _ in range(max_iter):
        idx = np.nonzero(active)[0]
        if idx.size == 0:
            break
        pa, sa = p[idx], sig[idx]
        g, H = _nh_grad_hess(pa, sa, k, mu, lam)
        gn = np.linalg.norm(g, axis=1)
        done = gn <= tol * k * scale[idx]
        active[idx[done]] = False
        keep = ~done
        idx, pa, sa, g, H = idx[keep], pa[keep], sa[keep], g[keep], H[keep]
        if idx.size == 0:
            break
        try:
            d = -np.linalg.solve(H, g[:, :, None])[:, :, 0]
        except np.linalg.LinAlgError:
            d = -g / (k + mu)
        bad = ((d * g).sum(1) >= 0) | ~np.all(np.isfinite(d), axis=1)
        d[bad] = -g[bad] / (k + mu)
        f0 = _nh_f(pa, sa, k, mu, lam)
        # rounding allowance of f in fp64 (magnitude of its terms)
        lnJ0 = np.log(np.prod(pa, axis=1))
        fr = 1e-13 * (k * (pa * pa + sa * sa).sum(1) + mu * (pa * pa).sum(1)
                      + mu * np.abs(lnJ0) + lam * lnJ0 * lnJ0 + mu)
        t = np.ones(idx.size)
        slope = (d * g).sum(1)
        for _ls in range(60):
            pn = pa + t[:, None] * d
            ok = np.all(pn > 0, axis=1)
            fn = np.full(idx.size, np.inf)
            fn[ok] = _nh_f(pn[ok], sa[ok], k, mu, lam)
            acc = ok & (fn <= f0 + 1e-4 * t * slope + fr)
            if np.all(acc):
                break
            t = np.where(acc, t, 0.5 * t)
        p[idx] = pa + t[:, None] * d
    return p


def project(F: np.ndarray, model: int, k: float, mu: float, lam: float):
    """p_i = U diag(p*) V^T  (eq. PD local; A5)."""
    U, s, V = signed_svd(F)
    ps = project_sigma(s, model, k, mu, lam)
    return np.einsum("tij,tj,tkj->tik", U, ps, V)


def elastic_forces(P: np.ndarray, F: np.ndarray, Bm: np.ndarray, w: np.ndarray, h: float,
                   T: np.ndarray, n_v: int):
    """sum_i h^2 w_i G_i^T (p_i - F_i) at vertex level, [n_v, 3]."""
    g = shape_gradients(Bm)
    Q = (h * h * w)[:, None, None] * (P - F)
    fv = np.einsum("tij,taj->tai", Q, g)       # [n_t, 4, 3]: Q g_a
    out = np.zeros((n_v, 3))
    np.add.at(out, T.reshape(-1), fv.reshape(-1, 3))
    return out


def gt_p(P: np.ndarray, Bm: np.ndarray, w: np.ndarray, h: float, T: np.ndarray, n_v: int):
    """sum_i h^2 w_i G_i^T p_i at vertex level (second term of b)."""
    g = shape_gradients(Bm)
    fv = np.einsum("tij,taj->tai", (h * h * w)[:, None, None] * P, g)
    out = np.zeros((n_v, 3))
    np.add.at(out, T.reshape(-1), fv.reshape(-1, 3))
    return out


# ---------------------------------------------------------------------------
# NCP functions (App. B.2, Fischer-Burmeister)
# ---------------------------------------------------------------------------
def fb_normal(y, lam_n, r):
    """phi_n = y + r lam - sqrt(y^2 + r^2 lam^2); theta_n = 1 - y/S;
    E_n = (1 - r lam/S) r.  S = 0 -> theta 1, E 0 (A15)."""
    y = np.asarray(y, dtype=np.float64)
    lam_n = np.asarray(lam_n, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    S = np.sqrt(y * y + r * r * lam_n * lam_n)
    pos = S > 0
    Ss = np.where(pos, S, 1.0)
    phi = np.where(pos, y + r * lam_n - S, 0.0)
    theta = np.where(pos, 1.0 - y / Ss, 1.0)
    E = np.where(pos, (1.0 - r * lam_n / Ss) * r, 0.0)
    return phi, theta, E


def fb_friction(ydot, lam_f, lam_n, mu, r):
    """theta_f, E_f for one contact's two friction rows.

    lam_n > 0 and mu lam_n > 0: theta_f = 1,
      E_f = r (R - r q) / (s + mu r lam_n - R), s = |ydot|, R = sqrt(s^2 + r^2 q^2),
      q = mu lam_n - min(|lam_f|, mu lam_n)   (reading A16c).
      The second argument of Coulomb's complementarity 0 <= |ydot_f| _|_ mu lam_n - |lam_f| >= 0
      (eq. coulomb's law 2) is evaluated at the projection of lam_f onto the cone: with
      the printed q = mu lam_n - |lam_f| the denominator equals phi_FB(s, q) + r |lam_f|, which
      vanishes at |lam_f| = 2 mu lam_n (s = 0) and is negative beyond it -- a pole and an
      anti-dissipative compliance at iterates outside the cone, reachable because lambda is not
      projected (A20).  Inside the cone (|lam_f| <= mu lam_n) the formula is the printed one; on
      and outside it q = 0, R = s and E_f = |ydot_f| / (mu lam_n), Coulomb's ratio
      |ydot_f| / |lam_f| on the cone boundary.  E_f is then continuous, >= 0 and bounded
      by r s / (r min(|lam_f|, mu lam_n)).  The only remaining 0/0 point is (s, |lam_f|) = (0, 0),
      where the limit is 0 (reading A16): E_f = 0 when the denominator is <= 1e-12 (s + mu r lam_n).
    otherwise (inactive, or degenerate cone mu lam_n = 0, reading A16b):
      theta_f = 0, E_f = 1 (identity), so lam_f -> 0.
    """
    ydot = np.asarray(ydot, dtype=np.float64)
    lam_f = np.asarray(lam_f, dtype=np.float64)
    s = np.linalg.norm(ydot, axis=-1)
    q = mu * lam_n - np.minimum(np.linalg.norm(lam_f, axis=-1), mu * lam_n)   # A16c
    R = np.sqrt(s * s + r * r * q * q)
    act = (lam_n > 0) & (mu * lam_n > 0)
    num = r * (R - r * q)
    den = s + mu * r * lam_n - R
    ok = den > 1e-12 * (s + mu * r * lam_n)                                       # A16
    with np.errstate(divide="ignore", invalid="ignore"):
        E = np.where(act, np.where(ok, num / np.where(ok, den, 1.0), 0.0), 1.0)
    theta = np.where(act, 1.0, 0.0)
    return theta, E


# ---------------------------------------------------------------------------
# NCP functions (App. B.1, minimum map) -- the ablation of P:L1200-1214 (NEXT row 1)
# ---------------------------------------------------------------------------
def minmap_normal(y, lam_n, r):
    """phi_n = y if y <= r lam else r lam;  theta_n = dphi/dy = 1 | 0;
    E_n = dphi/dlam = 0 | r."""
    y = np.asarray(y, dtype=np.float64)
    rl = np.asarray(r, dtype=np.float64) * np.asarray(lam_n, dtype=np.float64)
    first = y <= rl
    phi = np.where(first, y, rl)
    theta = np.where(first, 1.0, 0.0)
    E = np.where(first, 0.0, np.asarray(r, dtype=np.float64) * np.ones_like(y))
    return phi, theta, E


def minmap_friction(ydot, lam_f, lam_n, mu, r):
    """theta_f = [lam_n > 0]; E_f = identity if lam_n <= 0,
    0 if |ydot| <= r (mu lam_n - |lam_f|) (stick), else (|ydot| - r (mu lam_n - |lam_f|)) /
    (mu lam_n) (slip).  A degenerate cone mu lam_n <= 0 takes the inactive branch (reading
    A16b, as for FB); phi_f = theta_f ydot + E_f lam_f (reading A14)."""
    ydot = np.asarray(ydot, dtype=np.float64)
    lam_f = np.asarray(lam_f, dtype=np.float64)
    s = np.linalg.norm(ydot, axis=-1)
    q = mu * lam_n - np.linalg.norm(lam_f, axis=-1)
    act = (lam_n > 0) & (mu * lam_n > 0)
    stick = s <= r * q
    with np.errstate(divide="ignore", invalid="ignore"):
        slip = (s - r * q) / np.where(act, mu * lam_n, 1.0)
    E = np.where(act, np.where(stick, 0.0, slip), 1.0)
    theta = np.where(act, 1.0, 0.0)
    return theta, E


# ---------------------------------------------------------------------------
# Conjugate Residual (Saad, Iterative Methods, Alg. 6.20); reading A19
# ---------------------------------------------------------------------------
def cr_solve(apply, b: np.ndarray, n_iter: int, tiny: float = 1e-300):
    """Solve S z = b with z0 = 0 and exactly n_iter CR iterations (n_iter
    matvecs); stop early only on exact breakdown.  Returns (z, |r|)."""
    z = np.zeros_like(b)
    r = b.copy()
    if n_iter <= 0 or not np.any(r):
        return z, float(np.linalg.norm(r))
    Ar = apply(r)
    p = r.copy()
    Ap = Ar.copy()
    rAr = float(r @ Ar)
    for it in range(n_iter):
        ApAp = float(Ap @ Ap)
        if ApAp <= tiny or abs(rAr) <= tiny:
            break
        alpha = rAr / ApAp
        z += alpha * p
        r -= alpha * Ap
        if it == n_iter - 1:
            break
        Ar = apply(r)
        rAr_new = float(r @ Ar)
        beta = rAr_new / rAr
        rAr = rAr_new
        p = r + beta * p
        Ap = Ar + beta * Ap
    return z, float(np.linalg.norm(r))


# ---------------------------------------------------------------------------
# contact rows (App. A)
# ---------------------------------------------------------------------------
def gram_schmidt_tangents(n):
    """Tangents 'via the Gram-Schmidt process' (reading A13): e_a =
    axis least aligned with n (first on ties), t1 = normalize(e_a - (n.e_a) n),
    t2 = n x t1."""
    n = np.asarray(n, dtype=np.float64)
    e = np.zeros(3)
    e[int(np.argmin(np.abs(n)))] = 1.0
    t1 = e - np.dot(n, e) * n
    t1 = t1 / np.linalg.norm(t1)
    return t1, np.cross(n, t1)


@dataclasses.dataclass
class Rows:
    """Stacked constraint rows; row j = (c_j, vertices, weights) so that
    (J x)_j = c_j . sum_a w_ja x_a  (App. A)."""
    c: np.ndarray          # [m, 3]
    verts: np.ndarray      # [m, 4] int (padded with -1)
    wts: np.ndarray        # [m, 4]
    kind: np.ndarray       # [m] 0 normal, 1 friction, 2 bilateral
    contact: np.ndarray    # [m] owning contact index


def contact_rows(contacts):
    """Rows per contact: kind 0 -> (n, t1, t2); kind 1 -> (n) bilateral."""
    c, V, W, kind, own = [], [], [], [], []
    for j, ct in enumerate(contacts):
        vv = list(ct.verts) + [-1] * (4 - len(ct.verts))
        ww = list(ct.weights) + [0.0] * (4 - len(ct.weights))
        n = np.asarray(ct.normal, dtype=np.float64)
        if ct.kind == 1:
            dirs, kinds = [n], [2]
        else:
            t1, t2 = ct.tangent1, ct.tangent2
            if t1 is None or not np.any(t1):
                t1, t2 = gram_schmidt_tangents(n)
            dirs, kinds = [n, np.asarray(t1, float), np.asarray(t2, float)], [0, 1, 1]
        for d, kd in zip(dirs, kinds):
            c.append(d)
            V.append(vv)
            W.append(ww)
            kind.append(kd)
            own.append(j)
    if not c:
        return Rows(np.zeros((0, 3)), np.zeros((0, 4), int), np.zeros((0, 4)),
                    np.zeros(0, int), np.zeros(0, int))
    return Rows(np.asarray(c), np.asarray(V, dtype=np.int64), np.asarray(W),
                np.asarray(kind), np.asarray(own))


def carry_multipliers(old_contacts, old_lam, new_contacts):
    """lambda^0 for a new contact set (reading A10): Alg. 4 keeps lambda across frames
    (P:L939-961 never resets it); when collision detection produces a new set, each new
    contact keeps the rows of an identical constraint of the previous set -- same kind,
    vertices, weights and row directions (n, t1, t2); the first unused one in the previous
    order -- and starts from 0 otherwise."""
    ro, rn = contact_rows(old_contacts), contact_rows(new_contacts)
    lam = np.zeros(rn.c.shape[0])
    if old_lam is None or len(old_contacts) == 0:
        return lam
    old_lam = np.asarray(old_lam, dtype=np.float64)

    def starts(rows):
        out, j = [], 0
        while j < rows.c.shape[0]:
            n = 1 if rows.kind[j] == 2 else 3
            out.append((j, n))
            j += n
        return out

    def key(rows, j, n):
        return (n, rows.verts[j].tobytes(), rows.wts[j].tobytes(), rows.c[j:j + n].tobytes())

    pool = {}
    for j, n in starts(ro):
        pool.setdefault(key(ro, j, n), []).append(j)
    for j, n in starts(rn):
        cand = pool.get(key(rn, j, n))
        if cand:
            o = cand.pop(0)
            lam[j:j + n] = old_lam[o:o + n]
    return lam


# ---------------------------------------------------------------------------
# the frame loop (Alg. 4)
# ---------------------------------------------------------------------------
class Oracle:
    """fp64 Alg. 4 for one mesh.

    Vertex-level vectors are [n_v, 3]; the unknowns are the free vertices
    (Dirichlet pins by elimination, reading A7).
    """

    def __init__(self, mesh, material, h: float, lg_iters: int = 5,
                 cr_iters: Optional[int] = None, ncp: int = NCP_FB, precond: int = PRECOND_DELASSUS,
                 admm: bool = False, warm_start: bool = False):
        self.X = np.asarray(mesh.X, dtype=np.float64)
        self.len_scale = max(float(np.linalg.norm(self.X.max(0) - self.X.min(0))), float(np.abs(self.X).max()))
        self.T = np.asarray(mesh.T, dtype=np.int64)
        self.fixed = np.asarray(mesh.fixed).astype(bool)
        self.n_v = self.X.shape[0]
        self.h = float(h)
        self.model = int(material.model)
        self.mu, self.lam = lame(material.youngs, material.poisson)
        self.k = material.proj_stiffness if material.proj_stiffness > 0 else 2.0 * self.mu
        self.g = np.asarray(material.gravity, dtype=np.float64)
        self.lg_iters = int(lg_iters)
        self.cr_iters = int(material.cr_iterations if cr_iters is None else cr_iters)
        self.ncp = int(ncp)            # FB (the paper's choice) or min-map (App. B.1)
        self.precond = int(precond)    # Delassus diagonal (eq. complementarity preconditioner) or mass inverse
        # ADMM-PD (Overby et al. 2017; "our implementations are mainly based on PD and ADMM-PD",
        # P:L1340): per-tet dual u, reset to 0 each frame (reading A33)
        self.admm = bool(admm)
        # frame start (readings A9/A10 vs A9w/A10w)
        self.warm_start = bool(warm_start)
        self.Bm, self.vol, self.w, self.M = rest_data(self.X, self.T, material.density, self.k)
        self.A = assemble_Av(self.n_v, self.T, self.Bm, self.w, self.M, self.h)
        self.free = np.nonzero(~self.fixed)[0]
        self.pinned = np.nonzero(self.fixed)[0]
        A = self.A
        self.A_ff = A[self.free][:, self.free].tocsc()
        self.A_fc = A[self.free][:, self.pinned].tocsr()
        self.lu = spla.splu(self.A_ff)
        self.rows = None
        self.set_contacts([])

    # --- global step: x_f = A_ff^-1 b_f (3 RHS: A = A_v (x) I_3) -----------
    def solve(self, b_f: np.ndarray) -> np.ndarray:
        return self.lu.solve(np.ascontiguousarray(b_f))

    # --- per-contact setup (App. A) -------
    def set_contacts(self, contacts: List):
        self.contacts = list(contacts)
        self.rows = contact_rows(self.contacts)
        m = self.rows.c.shape[0]
        self.m = m
        if m == 0:
            self.D = np.zeros((0, 0))
            return
        pos = -np.ones(self.n_v, dtype=np.int64)
        pos[self.free] = np.arange(self.free.size)
        V, W = self.rows.verts, self.rows.wts
        if np.any(self.fixed[V[V >= 0]]):
            raise ValueError("contact on a pinned vertex")
        vc = np.unique(V[V >= 0])
        E = np.zeros((self.free.size, vc.size))
        E[pos[vc], np.arange(vc.size)] = 1.0
        Z = self.lu.solve(E)                   # A_v^-1 restricted to contact columns
        G = Z[pos[vc], :]                      # G[a,b] = (A_v^-1)_{ab}, a,b in V_c
        slot = {int(v): i for i, v in enumerate(vc)}
        # Wmat[j, s] = w_ja for the vertex in slot s
        Wm = np.zeros((m, vc.size))
        for j in range(m):
            for q in range(4):
                if V[j, q] >= 0:
                    Wm[j, slot[int(V[j, q])]] += W[j, q]
        C = self.rows.c
        # D = J A^-1 J^T, with A^-1 = A_v^-1 (x) I_3: D_jk = (c_j.c_k) (W G W^T)_jk
        self.D = (Wm @ G @ Wm.T) * (C @ C.T)
        self.G, self.vc, self.Wm = G, vc, Wm
        djj = np.diag(self.D).copy()
        kind = self.rows.kind
        if self.precond == PRECOND_MASS:
            # Macklin's choice: [J M^-1 J^T]_jj with the lumped M (A6), M = M_v (x) I_3
            Minv = 1.0 / self.M[vc]
            djj = (Wm * Wm) @ Minv * np.einsum("jd,jd->j", C, C)
        # preconditioner (P:L921-922 / P:L875-876): unilateral h^2 [.]_jj, frictional h [.]_jj
        self.r_row = np.where(kind == 1, self.h * djj, self.h * self.h * djj)
        own = self.rows.contact
        self.mu_c = np.array([ct.mu for ct in self.contacts], dtype=np.float64)
        self.d_row = np.zeros(m)
        for j in range(m):
            ct = self.contacts[own[j]]
            if kind[j] == 1:   # d_f = t . v_obstacle (A24)
                self.d_row[j] = float(np.dot(C[j], np.asarray(ct.obstacle_velocity, float)))
            else:
                self.d_row[j] = float(ct.offset)
        self.e_row = np.array([self.contacts[own[j]].compliance if kind[j] == 2 else 0.0
                               for j in range(m)])

    def Jx(self, x: np.ndarray) -> np.ndarray:
        """(J x)_j = c_j . sum_a w_ja x_a."""
        V, W = self.rows.verts, self.rows.wts
        xs = np.zeros((self.m, 3))
        for q in range(4):
            ok = V[:, q] >= 0
            xs[ok] += W[ok, q][:, None] * x[V[ok, q]]
        return np.einsum("jd,jd->j", self.rows.c, xs)

    def JT(self, lam_rows: np.ndarray) -> np.ndarray:
        """J^T v at vertex level, [n_v, 3]."""
        out = np.zeros((self.n_v, 3))
        V, W = self.rows.verts, self.rows.wts
        for q in range(4):
            ok = V[:, q] >= 0
            np.add.at(out, V[ok, q], (W[ok, q] * lam_rows[ok])[:, None] * self.rows.c[ok])
        return out

    # --- indicators (App. B.2) ------------------------------------
    def indicators(self, x, x_t, lam):
        """theta, E (per row), phi (per row: phi_n, phi_f components) and the
        Schur RHS pieces at x^k (reading A22)."""
        h = self.h
        kind, own = self.rows.kind, self.rows.contact
        Jx = self.Jx(x)
        Jxt = self.Jx(x_t)
        theta = np.ones(self.m)
        E = np.zeros(self.m)
        phi = np.zeros(self.m)
        ncont = len(self.contacts)
        # row index of each contact's normal / friction rows
        first = np.zeros(ncont, dtype=np.int64)
        seen = np.zeros(ncont, dtype=bool)
        for j in range(self.m):
            if not seen[own[j]]:
                first[own[j]] = j
                seen[own[j]] = True
        for cidx, ct in enumerate(self.contacts):
            j0 = first[cidx]
            if ct.kind == 1:
                theta[j0] = 1.0                       # A17
                E[j0] = self.e_row[j0]
                continue
            yn = Jx[j0] - self.d_row[j0]              # y_n = J_n x^k - d_n
            # reading A15: a gap within rounding of zero is zero.  At (y, lambda) = (0, 0) the
            # normal NCP's derivative theta_n = 1 - y/|y| jumps between 0 and 2 with the sign
            # of y, so the evaluation's own rounding must not pick the branch: the 0/0 rule
            # (theta_n = 1, E_n = 0) applies to every |y| <= 1e-12 L, L = max(rest bbox diagonal,
            # max |rest coordinate|) (the rounding of J_n x - d_n is ~1e-16 L)
            if abs(yn) <= 1e-12 * self.len_scale:
                yn = 0.0
            nfun, ffun = (minmap_normal, minmap_friction) if self.ncp == NCP_MINMAP else (fb_normal, fb_friction)
            ph, th, En = nfun(yn, lam[j0], self.r_row[j0])
            phi[j0], theta[j0], E[j0] = ph, th, En
            jf = [j0 + 1, j0 + 2]
            # h ydot_f = J_f (x^k - x_t) - h d_f
            ydot = (Jx[jf] - Jxt[jf]) / h - self.d_row[jf]
            thf, Ef = ffun(ydot, lam[jf], lam[j0], ct.mu, self.r_row[jf[0]])
            theta[jf] = thf
            E[jf] = Ef
            phi[jf] = thf * ydot + Ef * lam[jf]       # A14
        return theta, E, phi, Jx

    # --- one frame ------------------------------------------------------------
    def frame(self, x_t: np.ndarray, v_t: np.ndarray, pin_targets: Optional[np.ndarray] = None,
              capture: bool = False, lam0: Optional[np.ndarray] = None, start=None):
        """Alg. 4 body for one time step.  Returns (x, v, info); info["lam"] holds the
        multipliers at frame end.

        Default (readings A9, A10): x^0 = s, lambda^0 = 0; lam0 must be None.
        warm_start (A9w, A10w): x^0 = x_t + h v_t (the inertial extrapolation without the
        external-force term; s still enters b = M s + ...) and lambda^0 = lam0, the
        previous frame's final lambda (Alg. 4, never resets lambda inside
        `while simulation`; carried across a contact change by carry_multipliers), None = 0.
        start: (x_k, lambda_k, k) continues the frame from iterate k (the conditioning checks of
        tests/_parity.py); x_k must carry the pinned targets."""
        h = self.h
        x_t = np.asarray(x_t, dtype=np.float64)
        v_t = np.asarray(v_t, dtype=np.float64)
        # s = x_t + h v_t + h^2 M^-1 f_ext, f_ext = M g (A8)
        s = x_t + h * v_t + h * h * self.g[None, :]
        if lam0 is not None and not self.warm_start:
            raise ValueError("lam0 needs warm_start=True (reading A10: lambda^0 = 0)")
        x = x_t + h * v_t if self.warm_start else s.copy()   # x^0 (A9w / A9)
        if self.pinned.size:
            tgt = x_t[self.pinned] if pin_targets is None else np.asarray(pin_targets, float)
            x[self.pinned] = tgt
        lam = np.zeros(self.m) if lam0 is None else np.array(lam0, dtype=np.float64)   # lambda^0 (A10)
        if lam.shape != (self.m,):
            raise ValueError(f"lam0 must hold {self.m} rows")
        k0 = 0
        if start is not None:
            x, lam, k0 = np.array(start[0], dtype=np.float64), np.array(start[1], dtype=np.float64), int(start[2])
        F_ = self.free
        info = {"iters": [], "lam": None}
        u = np.zeros((self.T.shape[0], 3, 3))          # ADMM dual (reading A33)
        for it in range(k0, self.lg_iters):
            F = deformation_gradients(x, self.T, self.Bm)
            if self.admm:
                # ADMM-PD: z = argmin psi(z) + w/2 |F + u - z|^2; u <- u + F - z;
                # the global step targets z - u (Overby et al. 2017, Alg. 1)
                P = project(F + u, self.model, self.k, self.mu, self.lam)
                u = u + F - P
                target = P - u
            else:
                P = project(F, self.model, self.k, self.mu, self.lam)
                target = P
            # b = M s + h^2 sum w G^T p - A_fc x_c  (A7)
            b = self.M[:, None] * s + gt_p(target, self.Bm, self.w, h, self.T, self.n_v)
            b_f = b[F_]
            if self.pinned.size:
                b_f = b_f - self.A_fc @ x[self.pinned]
            rec = {}
            if capture:
                r_f = b_f - self.A_ff @ x[F_]
                rec.update(F=F, P=P, b_f=b_f.copy(), resid=r_f)
            if self.m == 0:
                xn = x.copy()
                xn[F_] = self.solve(b_f)               # x^{k+1} = A^-1 b
            else:
                theta, E, phi, Jx = self.indicators(x, x_t, lam)
                kind = self.rows.kind
                # g = b + h^2 H^T lambda^k, H = Theta J
                g_f = b_f + h * h * self.JT(theta * lam)[F_]
                xt_f = self.solve(g_f)
                xt = x.copy()
                xt[F_] = xt_f
                # h-vector
                hvec = np.where(kind == 2, self.d_row - E * lam,
                                np.where(kind == 0, -phi + theta * Jx, -h * phi + theta * Jx))
                rho = hvec - theta * self.Jx(xt)       # h - H A^-1 g (Alg. 3/4 sign, A11)
                Cdiag = np.where(kind == 1, E / h, E / (h * h))   # C
                S_apply = lambda v: theta * (self.D @ (theta * v)) + Cdiag * v
                z, res = cr_solve(S_apply, rho, self.cr_iters)
                lam = lam + z / (h * h)                # Delta lambda = z / h^2 (A11), no projection (A20)
                # x^{k+1} = A^-1 (b + h^2 H^T lambda^{k+1})
                xn = x.copy()
                xn[F_] = self.solve(b_f + h * h * self.JT(theta * lam)[F_])
                info["theta_last"] = theta
                if capture:
                    rec.update(theta=theta, E=E, phi=phi, rho=rho, z=z, cr_res=res,
                               x_tilde=xt)
            if capture:
                rec["x_next"] = xn.copy()
                rec["lam"] = lam.copy()
                info["iters"].append(rec)
            x = xn
        info["lam"] = lam
        v = (x - x_t) / h
        return x, v, info

    # --- frame-end classification (A21) --------------------------------------
    def classify(self, x, x_t, lam):
        """Per unilateral contact: 0 inactive, 1 stick, 2 slip (reading A21)."""
        out = []
        Jx, Jxt = self.Jx(x), self.Jx(x_t)
        j = 0
        for ct in self.contacts:
            if ct.kind == 1:
                j += 1
                out.append(-1)
                continue
            ln = lam[j]
            jf = [j + 1, j + 2]
            ydot = (Jx[jf] - Jxt[jf]) / self.h - self.d_row[jf]
            if not ln > 0:
                out.append(0)
            else:
                q = ct.mu * ln - np.linalg.norm(lam[jf])
                out.append(1 if np.linalg.norm(ydot) <= self.r_row[jf[0]] * q else 2)
            j += 3
        return np.asarray(out)
