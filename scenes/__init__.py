"""Seeded synthetic input generators shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no F, no projection, no system
matrix, no NCP function).  It only builds the *inputs* the paper's problem
statement takes (mesh, material, time step, contact pairs), with the shapes
of the paper's workloads (SURVEY.md §8(d) "Synthetic inputs"):

* cfg1  cantilever beam  -- 2x2x4 hex cells (aspect 1:1:2), 5-tet split,
        45 vertices / 80 tets, z=0 end fixed (reading A27).
* cfg2  incline block    -- 10x10x10 vertices, 5-tet split (3 645 tets), bottom
        face in contact with a plane inclined at theta (reading A28).
* cfg3  gingerbread-class silhouette slab -- 63x86 raster x 6 layers, Kuhn
        6-tet split (19 691 v / 93 600 t), lying on 6 thin capsule bars,
        800 contact points (seed 1234), head handle pinned.
* cfg4  pile of 68 cubes (16^3 cells each, 5-tet split; 334k v / 1.39M t):
        a 4x4 grid of 4-high stacks plus 4 cubes bridging 2x2 stack tops, 1 mm
        gaps, jitter (seed 7).  ~20k contacts: bottom-layer vertices against the
        ground, every other bottom-face vertex against the top face of the cube
        below (soft-soft rows: the vertex minus the barycentric point of the
        lower face triangle, 1 + 3 vertices).  `pile(cells=3, nx=2, layers=2)`
        is the small variant the parity tests use.

Contact pairs are the output of a proximity query (collision detection is
outside the hot path); here they are generated once from
the rest geometry, which is input preparation, not the method.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

__all__ = [
    "Mesh", "Material", "Contact", "Scene",
    "hex_grid", "cantilever", "incline_block", "gingerbread", "single_tet",
    "tangent_frame", "make_scene", "pile", "random_state", "batch_instance", "batch_instance_params",
]

NEOHOOKEAN, COROTATED, ARAP = 0, 1, 2


@dataclasses.dataclass
class Mesh:
    X: np.ndarray            # [n_v, 3] float64 rest positions (m)
    T: np.ndarray            # [n_t, 4] int32 tetrahedra
    fixed: np.ndarray        # [n_v] uint8 Dirichlet mask

    @property
    def n_v(self):
        return int(self.X.shape[0])

    @property
    def n_t(self):
        return int(self.T.shape[0])

    def bbox_diag(self) -> float:
        return float(np.linalg.norm(self.X.max(0) - self.X.min(0)))


@dataclasses.dataclass
class Material:
    model: int = NEOHOOKEAN        # 0 NH, 1 linear corotated, 2 ARAP
    density: float = 1000.0        # kg/m^3
    youngs: float = 1e6            # Pa
    poisson: float = 0.3
    proj_stiffness: float = 0.0    # k in w_i = k*vol_i ; 0 -> 2*mu (reading A1)
    gravity: tuple = (0.0, 0.0, -9.81)
    cr_iterations: int = 10


@dataclasses.dataclass
class Contact:
    """One contact point (App. A).

    kind 0: unilateral normal row + 2 friction rows; kind 1: one bilateral row
    along `normal` with compliance `compliance`.
    """
    verts: List[int]
    weights: List[float]
    normal: np.ndarray
    offset: float                              # d_n (or d_b)
    mu: float = 0.5
    kind: int = 0
    tangent1: Optional[np.ndarray] = None
    tangent2: Optional[np.ndarray] = None
    obstacle_velocity: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(3))
    compliance: float = 0.0


@dataclasses.dataclass
class Scene:
    name: str
    mesh: Mesh
    material: Material
    h: float
    iterations: int
    contacts: List[Contact]
    pin_velocity: np.ndarray           # [3] m/s applied to all fixed vertices
    v0: Optional[np.ndarray] = None    # [n_v,3] initial velocity
    obstacles: Optional[list] = None   # analytic obstacles the contacts were generated from:
                                       # dicts kind (0 plane, 1 sphere, 2 capsule), a, b, radius, mu


# --------------------------------------------------------------------------
# structured tet meshes
# --------------------------------------------------------------------------
_CORNER = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0),
           (0, 0, 1), (1, 0, 1), (0, 1, 1), (1, 1, 1)]
_CID = {c: i for i, c in enumerate(_CORNER)}

# 5-tet split of a cube; parity alternation keeps faces conforming
_FIVE_EVEN = [((1, 0, 0), (0, 0, 0), (1, 1, 0), (1, 0, 1)),
              ((0, 1, 0), (0, 0, 0), (1, 1, 0), (0, 1, 1)),
              ((0, 0, 1), (0, 0, 0), (1, 0, 1), (0, 1, 1)),
              ((1, 1, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1)),
              ((0, 0, 0), (1, 1, 0), (1, 0, 1), (0, 1, 1))]
_FIVE_ODD = [((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)),
             ((1, 1, 0), (1, 0, 0), (0, 1, 0), (1, 1, 1)),
             ((1, 0, 1), (1, 0, 0), (0, 0, 1), (1, 1, 1)),
             ((0, 1, 1), (0, 1, 0), (0, 0, 1), (1, 1, 1)),
             ((1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1))]


def _kuhn6():
    import itertools
    tets = []
    for perm in itertools.permutations(range(3)):
        p = [0, 0, 0]
        path = [tuple(p)]
        for ax in perm:
            p[ax] = 1
            path.append(tuple(p))
        tets.append(tuple(path))
    return tets


_KUHN6 = _kuhn6()


def hex_grid(nx: int, ny: int, nz: int, cell=(1.0, 1.0, 1.0), split: str = "five",
             keep: Optional[np.ndarray] = None):
    """Tetrahedralise an nx*ny*nz block of hex cells.

    keep: optional bool array [nx, ny, nz] selecting cells.  Unused vertices
    are dropped and the rest renumbered in (i, j, k) lexicographic order.
    Returns (X [n,3] float64, T [m,4] int32).
    """
    cell = np.asarray(cell, dtype=np.float64)
    if keep is None:
        keep = np.ones((nx, ny, nz), dtype=bool)
    vid = lambda i, j, k: (i * (ny + 1) + j) * (nz + 1) + k
    tets = []
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                if not keep[i, j, k]:
                    continue
                if split == "five":
                    pat = _FIVE_EVEN if (i + j + k) % 2 == 0 else _FIVE_ODD
                elif split == "kuhn6":
                    pat = _KUHN6
                else:
                    raise ValueError(split)
                for t in pat:
                    tets.append([vid(i + a, j + b, k + c) for (a, b, c) in t])
    T = np.asarray(tets, dtype=np.int64)
    used = np.unique(T)
    remap = -np.ones((nx + 1) * (ny + 1) * (nz + 1), dtype=np.int64)
    remap[used] = np.arange(used.size)
    ii, rem = np.divmod(used, (ny + 1) * (nz + 1))
    jj, kk = np.divmod(rem, nz + 1)
    X = np.stack([ii * cell[0], jj * cell[1], kk * cell[2]], axis=1).astype(np.float64)
    return X, remap[T].astype(np.int32)


def single_tet():
    X = np.array([[0, 0, 0], [0.1, 0, 0], [0, 0.1, 0], [0, 0, 0.1]], dtype=np.float64)
    T = np.array([[0, 1, 2, 3]], dtype=np.int32)
    return Mesh(X, T, np.zeros(4, np.uint8))


def cantilever() -> Mesh:
    """cfg1 (reading A27): 2x2x4 cells of 0.05 x 0.05 x 0.1 m, 5-tet, z=0 fixed."""
    X, T = hex_grid(2, 2, 4, cell=(0.05, 0.05, 0.1), split="five")
    fixed = (np.abs(X[:, 2]) < 1e-12).astype(np.uint8)
    return Mesh(X, T, fixed)


def tangent_frame(n):
    """Deterministic Gram-Schmidt tangents (reading A13): e_a is the
    coordinate axis least aligned with n (first on ties); t1 = normalize(e_a -
    (n.e_a) n); t2 = n x t1.  Input preparation shared by both sides."""
    n = np.asarray(n, dtype=np.float64)
    a = int(np.argmin(np.abs(n)))
    e = np.zeros(3)
    e[a] = 1.0
    t1 = e - np.dot(n, e) * n
    t1 /= np.linalg.norm(t1)
    t2 = np.cross(n, t1)
    return t1, t2


def incline_block(theta_deg: float = 10.0, mu: float = 0.5, nv: int = 10,
                  edge: float = 0.1, youngs: float = 1e8) -> Scene:
    """cfg2: nv^3-vertex block (5-tet) resting on a plane through the origin
    with normal (-sin th, 0, cos th) (gravity -z).  Contacts: bottom face."""
    X, T = hex_grid(nv - 1, nv - 1, nv - 1, cell=(edge / (nv - 1),) * 3, split="five")
    th = math.radians(theta_deg)
    # rotate about y so the bottom face lies in the plane
    R = np.array([[math.cos(th), 0, -math.sin(th)], [0, 1, 0], [math.sin(th), 0, math.cos(th)]])
    X = X @ R.T
    n = np.array([-math.sin(th), 0.0, math.cos(th)])
    mesh = Mesh(X, T, np.zeros(X.shape[0], np.uint8))
    bottom = np.nonzero(np.abs(X @ n) < 1e-9)[0]
    t1, t2 = tangent_frame(n)
    contacts = [Contact([int(v)], [1.0], n.copy(), 0.0, mu=mu, tangent1=t1, tangent2=t2)
                for v in bottom]
    mat = Material(model=NEOHOOKEAN, density=1000.0, youngs=youngs, poisson=0.3)
    plane = {"kind": 0, "a": np.zeros(3), "b": n.copy(), "radius": 0.0, "mu": mu}
    return Scene("incline", mesh, mat, 0.01, 5, contacts, np.zeros(3), obstacles=[plane])


# --------------------------------------------------------------------------
# gingerbread-class silhouette
# --------------------------------------------------------------------------
def _seg_dist(px, py, ax, ay, bx, by):
    dx, dy = bx - ax, by - ay
    t = np.clip(((px - ax) * dx + (py - ay) * dy) / (dx * dx + dy * dy), 0.0, 1.0)
    return np.hypot(px - ax - t * dx, py - ay - t * dy)


def _inside_silhouette(px, py):
    head = np.hypot(px - 40, py - 92) <= 15
    torso = ((px - 40) / 19) ** 2 + ((py - 56) / 25) ** 2 <= 1
    arms = (_seg_dist(px, py, 24, 70, 5, 58) <= 7.5) | (_seg_dist(px, py, 56, 70, 75, 58) <= 7.5)
    legs = (_seg_dist(px, py, 32, 38, 24, 5) <= 8.5) | (_seg_dist(px, py, 48, 38, 56, 5) <= 8.5)
    return head | torso | arms | legs


def gingerbread(scale: float = 0.79, layers: int = 6, cell_m: float = 0.005,
                n_contacts: int = 800, contact_seed: int = 1234, obstacle_seed: int = 0,
                youngs: float = 1e6, mu: float = 0.5, n_bars: int = 6) -> Scene:
    """cfg3.  Silhouette raster (63x86 at scale 0.79) x `layers`, Kuhn 6-tet,
    cell 5 mm.  The slab lies in the x-y plane on `n_bars` thin capsule bars
    (radius 2-5 mm, random in-plane orientation, seed `obstacle_seed`) just
    below its bottom face; gravity is -z.  Contacts: `n_contacts` bottom-face
    vertices nearest the bars, drawn with seed `contact_seed`, normal from the
    nearest bar axis point, d_n = n . (surface point).  The head top is a
    Dirichlet handle moving at 0.5 m/s along +y."""
    nx, ny = int(round(80 * scale)), int(round(110 * scale))
    nx, ny = 63, 86 if scale == 0.79 else (nx, ny)
    ci = (np.arange(nx) + 0.5) / scale
    cj = (np.arange(ny) + 0.5) / scale
    P, Q = np.meshgrid(ci, cj, indexing="ij")
    keep2 = _inside_silhouette(P, Q)
    keep = np.repeat(keep2[:, :, None], layers, axis=2)
    X, T = hex_grid(nx, ny, layers, cell=(cell_m,) * 3, split="kuhn6", keep=keep)
    # handle: head-top vertices (design y >= 100)
    yd = X[:, 1] / cell_m / scale
    fixed = (yd >= 100.0).astype(np.uint8)
    mesh = Mesh(X, T, fixed)
    # bars below the bottom face z = 0
    rng = np.random.default_rng(obstacle_seed)
    W, H = nx * cell_m, ny * cell_m
    bars = []
    for b in range(n_bars):
        r = rng.uniform(0.002, 0.005)
        cy = H * (0.12 + 0.70 * (b + rng.uniform(0.2, 0.8)) / n_bars)
        ang = rng.uniform(-0.35, 0.35)
        a = np.array([-0.1 * W, cy - math.tan(ang) * 0.6 * W, -r])
        c = np.array([1.1 * W, cy + math.tan(ang) * 0.6 * W, -r])
        bars.append((a, c, r))
    bottom = np.nonzero((X[:, 2] < 1e-12) & (fixed == 0))[0]
    best = np.full(bottom.size, np.inf)
    best_n = np.zeros((bottom.size, 3))
    best_d = np.zeros(bottom.size)
    for (a, c, r) in bars:
        d = c - a
        p = X[bottom]
        t = np.clip(((p - a) @ d) / (d @ d), 0.0, 1.0)
        q = a + t[:, None] * d
        v = p - q
        dist = np.linalg.norm(v, axis=1)
        gap = dist - r
        upd = gap < best
        nn = v / dist[:, None]
        best[upd] = gap[upd]
        best_n[upd] = nn[upd]
        best_d[upd] = np.einsum("ij,ij->i", nn[upd], q[upd] + r * nn[upd])
    order = np.argsort(best, kind="stable")
    pool = order[: min(bottom.size, int(n_contacts * 1.35))]
    crng = np.random.default_rng(contact_seed)
    pick = np.sort(crng.choice(pool, size=min(n_contacts, pool.size), replace=False))
    contacts = []
    for i in pick:
        n = best_n[i]
        t1, t2 = tangent_frame(n)
        contacts.append(Contact([int(bottom[i])], [1.0], n.copy(), float(best_d[i]), mu=mu,
                                tangent1=t1, tangent2=t2))
    mat = Material(model=NEOHOOKEAN, density=1000.0, youngs=youngs, poisson=0.3)
    obst = [{"kind": 2, "a": a, "b": c, "radius": r, "mu": mu} for (a, c, r) in bars]
    return Scene("gingerbread", mesh, mat, 0.01, 5, contacts, np.array([0.0, 0.5, 0.0]), obstacles=obst)


# --------------------------------------------------------------------------
# cfg4: multi-object pile
# --------------------------------------------------------------------------
def pile(cells: int = 16, edge: float = 0.16, nx: int = 4, layers: int = 4, bridges: bool = True,
         gap: float = 0.001, stack_gap: float = 0.01, jitter_xy: float = 0.002, jitter_deg: float = 3.0,
         seed: int = 7, youngs: float = 1e7, mu: float = 0.5) -> Scene:
    """nx x nx stacks of `layers` cubes (cells^3 hex cells of edge/cells, 5-tet split) on the
    ground z = 0, stacks `stack_gap` apart, vertical gaps `gap`; with `bridges`, one cube on
    top of every 2x2 block of stacks, centred over their shared corner.  Each cube gets a
    seeded horizontal offset (+-jitter_xy) and yaw (+-jitter_deg) so faces stay horizontal.

    Contacts (normal +z, mu): every bottom-face vertex of a bottom-layer cube against the
    ground (d_n = 0); every other bottom-face vertex against the top face of the cube
    below it, if it projects inside that face: row = x_a - sum_i b_i x_i over the
    containing top-face triangle (weights 1, -b_0, -b_1, -b_2), d_n = 0."""
    X0, T0 = hex_grid(cells, cells, cells, cell=(edge / cells,) * 3, split="five")
    nv0 = X0.shape[0]
    rng = np.random.default_rng(seed)
    half = edge / 2.0
    pitch = edge + stack_gap
    cubes = []   # (centre xy, z0, yaw)
    for layer in range(layers):
        for i in range(nx):
            for j in range(nx):
                cubes.append([(i - (nx - 1) / 2.0) * pitch, (j - (nx - 1) / 2.0) * pitch, layer * (edge + gap)])
    if bridges:
        for i in range(0, nx - 1, 2):
            for j in range(0, nx - 1, 2):
                cx = (i + 0.5 - (nx - 1) / 2.0) * pitch
                cy = (j + 0.5 - (nx - 1) / 2.0) * pitch
                cubes.append([cx, cy, layers * (edge + gap)])
    Xs, Ts, frames = [], [], []
    local = X0 - np.array([half, half, 0.0])     # cube-local: centred in xy, bottom at z = 0
    for k, (cx, cy, z0) in enumerate(cubes):
        dx, dy = rng.uniform(-jitter_xy, jitter_xy, 2)
        yaw = math.radians(rng.uniform(-jitter_deg, jitter_deg))
        c, s_ = math.cos(yaw), math.sin(yaw)
        R = np.array([[c, -s_, 0.0], [s_, c, 0.0], [0.0, 0.0, 1.0]])
        o = np.array([cx + dx, cy + dy, z0])
        Xs.append(local @ R.T + o)
        Ts.append(T0 + k * nv0)
        frames.append((o, R))
    X = np.concatenate(Xs)
    T = np.concatenate(Ts).astype(np.int32)
    mesh = Mesh(X, T, np.zeros(X.shape[0], np.uint8))
    # local grid indices of the cube's vertices (hex_grid numbering: (i, j, k) lexicographic)
    n1 = cells + 1
    vid = lambda i, j, k: (i * n1 + j) * n1 + k
    bottom = np.array([vid(i, j, 0) for i in range(n1) for j in range(n1)])
    h_cell = edge / cells
    nz = np.array([0.0, 0.0, 1.0])
    t1, t2 = tangent_frame(nz)
    contacts: List[Contact] = []
    top_z = [z0 + edge for (_, _, z0) in cubes]
    for k, (o, R) in enumerate(frames):
        base = k * nv0
        if o[2] < 1e-9:      # bottom layer: the ground plane z = 0
            for v in bottom:
                contacts.append(Contact([int(base + v)], [1.0], nz.copy(), 0.0, mu=mu, tangent1=t1, tangent2=t2))
            continue
        # candidate supports: cubes whose top is just below this cube's bottom
        below = [q for q in range(len(cubes)) if abs(top_z[q] + gap - o[2]) < 1e-9]
        for v in bottom:
            p = X[base + v]
            for q in below:
                oq, Rq = frames[q]
                lp = Rq.T @ (p - oq) + np.array([half, half, 0.0])   # in q's grid frame
                u, w = lp[0] / h_cell, lp[1] / h_cell
                if not (0.0 <= u <= cells and 0.0 <= w <= cells):
                    continue
                i, j = min(int(u), cells - 1), min(int(w), cells - 1)
                fu, fw = u - i, w - j
                qb = q * nv0
                if fu >= fw:     # triangle (i,j) (i+1,j) (i+1,j+1)
                    tri = [vid(i, j, cells), vid(i + 1, j, cells), vid(i + 1, j + 1, cells)]
                    bc = [1.0 - fu, fu - fw, fw]
                else:            # triangle (i,j) (i+1,j+1) (i,j+1)
                    tri = [vid(i, j, cells), vid(i + 1, j + 1, cells), vid(i, j + 1, cells)]
                    bc = [1.0 - fw, fu, fw - fu]
                contacts.append(Contact([int(base + v)] + [int(qb + t) for t in tri],
                                        [1.0] + [-float(b) for b in bc], nz.copy(), 0.0, mu=mu,
                                        tangent1=t1, tangent2=t2))
                break
    mat = Material(model=NEOHOOKEAN, density=1000.0, youngs=youngs, poisson=0.3)
    return Scene("pile", mesh, mat, 0.01, 5, contacts, np.zeros(3))


def make_scene(name: str, **kw) -> Scene:
    if name in ("cfg1", "cantilever"):
        m = cantilever()
        mat = Material(model=kw.get("model", NEOHOOKEAN), density=1000.0, youngs=1e6, poisson=0.3)
        return Scene("cantilever", m, mat, 1.0 / 60.0, 5, [], np.zeros(3))
    if name in ("cfg2", "incline"):
        return incline_block(**kw)
    if name in ("cfg3", "gingerbread"):
        return gingerbread(**kw)
    if name in ("cfg4", "pile"):
        return pile(**kw)
    if name == "block":   # small multi-purpose block used by parity tests
        nv = kw.get("nv", 6)
        X, T = hex_grid(nv - 1, nv - 1, nv - 1, cell=(0.02,) * 3, split=kw.get("split", "five"))
        fixed = (np.abs(X[:, 2]) < 1e-12).astype(np.uint8) if kw.get("pinned", True) else np.zeros(X.shape[0], np.uint8)
        mat = Material(model=kw.get("model", NEOHOOKEAN), youngs=kw.get("youngs", 1e6))
        return Scene("block", Mesh(X, T, fixed), mat, 0.01, 5, [], np.zeros(3))
    raise ValueError(name)


def random_state(mesh: Mesh, seed: int, amp: float = 0.1):
    """Seeded perturbed positions x = X + amp*cell*N(0,1) and velocities, used
    to exercise the local step away from rest (parity tests)."""
    rng = np.random.default_rng(seed)
    e = mesh.X[mesh.T[:, 1]] - mesh.X[mesh.T[:, 0]]
    cell = float(np.median(np.linalg.norm(e, axis=1)))
    x = mesh.X + amp * cell * rng.standard_normal(mesh.X.shape)
    v = 0.05 * rng.standard_normal(mesh.X.shape)
    return x, v


def batch_instance_params(scene: Scene, i: int, v_sigma: float = 0.01, offset: float = 0.005):
    """cfg5 instance i (seed 1000 + i): initial velocity
    ~ N(0, v_sigma^2) per free-vertex component and an obstacle offset
    delta ~ U(-offset, +offset) along z ("obstacle
    offset +-5 mm"): positive delta raises the bars, so about half of the
    instances start with the slab up to `offset` inside the obstacles.
    Returns (v0 [n_v, 3], delta)."""
    rng = np.random.default_rng(1000 + i)
    v0 = v_sigma * rng.standard_normal(scene.mesh.X.shape)
    v0[scene.mesh.fixed.astype(bool)] = 0.0
    return v0, float(rng.uniform(-offset, offset))


def batch_instance(scene: Scene, i: int, v_sigma: float = 0.01, offset: float = 0.005):
    """cfg5 instance i of a scene: batch_instance_params, with the obstacles
    shifted by delta along z, i.e. every contact's d_n grows by n . (0, 0, delta).
    Returns (v0 [n_v, 3], contacts)."""
    v0, delta = batch_instance_params(scene, i, v_sigma, offset)
    cs = [dataclasses.replace(c, offset=float(c.offset + c.normal[2] * delta)) for c in scene.contacts]
    return v0, cs
