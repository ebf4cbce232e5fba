"""CPU-only checks of the C-ABI library: it loads, exports every symbol the
header declares, validates its inputs, and its host precompute (ordering,
etree, Cholesky, K = L^-1) satisfies Theorem 1 and K^T K = A^-1 against the
oracle's independent dense solve.  No GPU compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

import scenes
from oracle import oracle as O
from paper_2503_15078_b200 import EXPORTED_SYMBOLS, Sim, SimError, lib, lib_path

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sim.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char \*)\s*\*?\s*(sim_\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    so = ctypes.CDLL(lib_path)
    for name in declared:
        assert hasattr(so, name), name
    assert declared == set(EXPORTED_SYMBOLS)


def _host(sc, **kw):
    return Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, host_only=True, **kw)


def _dense_K(s):
    perm, parent, rowptr, vals = s.debug_inverse()
    nf = perm.size
    first = np.arange(nf) - (rowptr[1:] - rowptr[:-1]) + 1
    K = np.zeros((nf, nf))
    for i in range(nf):
        K[i, first[i]:i + 1] = vals[rowptr[i]:rowptr[i + 1]]
    return perm, parent, first, K


@pytest.mark.parametrize("name,kw", [("cfg1", {}), ("block", {"nv": 5, "split": "kuhn6"}),
                                     ("block", {"nv": 4, "pinned": False})])
def test_sparse_inverse_theorem1_and_exactness(name, kw):
    """Thm 1: pattern(L^-1) = ancestor closure of the etree;
    postorder makes row i the contiguous range [first(i), i]; K^T K = A^-1
     to fp32 storage rounding, against the oracle's dense inverse."""
    sc = scenes.make_scene(name, **kw)
    s = _host(sc)
    perm, parent, first, K = _dense_K(s)
    nf = perm.size
    assert np.all((parent > np.arange(nf)) | (parent == -1))
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    pos = {int(v): k for k, v in enumerate(o.free)}
    idx = np.array([pos[int(p)] for p in perm])
    A = o.A_ff.toarray()[np.ix_(idx, idx)]
    Ainv = np.linalg.inv(A)
    assert np.abs(K.T @ K - Ainv).max() <= 2e-6 * np.abs(Ainv).max()
    Kd = np.linalg.inv(np.linalg.cholesky(A))
    anc = np.zeros((nf, nf), bool)
    for j in range(nf):
        i = j
        while i != -1:
            anc[i, j] = True
            i = parent[i]
    assert np.array_equal(np.abs(Kd) > 1e-13 * np.abs(Kd).max(), anc)
    # subtree of i is exactly [first(i), i] in postorder
    for i in range(nf):
        assert np.array_equal(np.nonzero(anc[i])[0], np.arange(first[i], i + 1))


def test_drop_tolerance_zeroes_small_entries():
    sc = scenes.make_scene("block", nv=5)
    _, _, _, K0 = _dense_K(_host(sc))
    _, _, _, K1 = _dense_K(_host(sc, drop_tolerance=1e-2))
    dropped = (K1 == 0) & (K0 != 0)
    assert dropped.any()
    diag = np.abs(np.diag(K0))
    assert np.all(np.abs(K0[dropped]) < 1e-2 * diag[np.nonzero(dropped)[1]] * 1.0001)


def test_drop_tolerance_shrinks_kpass_streams():
    """Reading A25 storage: each row's stored range starts at its first kept column, so dropped
    leading entries leave the K-pass tile streams (sim_stats.kpass_bytes, nnz_K_kept) while the
    kept entries stay exactly those of the exact K."""
    sc = scenes.make_scene("cfg3")
    st = {}
    for tol in (0.0, 1e-3, 1e-2):
        st[tol] = _host(sc, drop_tolerance=tol).stats()
    assert st[0.0]["nnz_K_kept"] == st[0.0]["nnz_K"]
    assert st[1e-2]["nnz_K_kept"] < st[1e-3]["nnz_K_kept"] < st[0.0]["nnz_K_kept"]
    assert st[1e-2]["kpass_bytes"] < st[1e-3]["kpass_bytes"] <= st[0.0]["kpass_bytes"]


def test_input_validation():
    sc = scenes.make_scene("cfg1")
    bad = scenes.Material(poisson=0.5)
    with pytest.raises(SimError, match="poisson"):
        _host(scenes.Scene("x", sc.mesh, bad, sc.h, 5, [], np.zeros(3)))
    T = sc.mesh.T.copy()
    T[3] = [0, 0, 1, 2]
    with pytest.raises(SimError, match="degenerate"):
        Sim(sc.mesh.X, T, sc.mesh.fixed, sc.material, sc.h, host_only=True)
    with pytest.raises(SimError, match="h must"):
        Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, -1.0, host_only=True)


def test_binding_checks_array_sizes():
    """The binding refuses arrays that do not hold n_instances x n_vertices x 3 values before the
    C call (the ABI trusts the caller's sizes)."""
    sc = scenes.make_scene("cfg1")
    s = _host(sc)
    with pytest.raises(ValueError, match="x must hold"):
        s.set_state(sc.mesh.X[:-1], np.zeros_like(sc.mesh.X))
    with pytest.raises(ValueError, match="b must hold"):
        s.debug_apply_inverse(np.zeros((sc.mesh.n_v + 1, 3)))
    with pytest.raises(ValueError, match="out must be"):
        s.get_positions(out=np.empty((1, sc.mesh.n_v, 3), np.float32))


def test_no_cpu_fallback_without_device():
    """sim_create (device path) must fail loudly when there is no GPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sc = scenes.make_scene("cfg1")
    with pytest.raises(SimError, match="CUDA"):
        Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h)


def test_cfg3_structure():
    """cfg3 gingerbread-class scene: sizes of SURVEY §8 (19 691 v / 93 600 t);
    K stays values-only (nnz = sum of subtree sizes)."""
    sc = scenes.make_scene("cfg3")
    assert sc.mesh.n_v == 19691 and sc.mesh.n_t == 93600 and len(sc.contacts) == 800
    s = _host(sc)
    st = s.stats()
    assert st["n_free"] == 19691 - int(sc.mesh.fixed.sum())
    assert 1.0e7 < st["nnz_K"] < 2.5e7


def test_forest_of_objects_sparse_inverse():
    """Several disconnected objects (SURVEY §8(d) cfg4 structure): the ordering dissects each
    connected component separately, the etree is a forest (one root per object), the Cholesky
    factorises the trees in parallel, and K^T K = A^-1 with K block-diagonal (Theorem 1)."""
    X, T = scenes.hex_grid(3, 3, 3, cell=(0.02,) * 3)
    n = X.shape[0]
    X3 = np.concatenate([X, X + [0.1, 0.0, 0.0], X + [0.0, 0.1, 0.01]])
    T3 = np.concatenate([T, T + n, T + 2 * n]).astype(np.int32)
    mesh = scenes.Mesh(X3, T3, np.zeros(X3.shape[0], np.uint8))
    mat = scenes.Material()
    s = Sim(mesh.X, mesh.T, mesh.fixed, mat, 0.01, host_only=True)
    perm, parent, rowptr, vals = s.debug_inverse()
    nf = perm.size
    assert np.sum(parent == -1) == 3
    first = np.arange(nf) - (rowptr[1:] - rowptr[:-1]) + 1
    K = np.zeros((nf, nf))
    for i in range(nf):
        K[i, first[i]:i + 1] = vals[rowptr[i]:rowptr[i + 1]]
    obj = perm // n                       # object of each internal index
    assert np.all((K == 0) | (obj[:, None] == obj[None, :]))
    o = O.Oracle(mesh, mat, 0.01)
    A = o.A_ff.toarray()[np.ix_(perm, perm)]
    Ainv = np.linalg.inv(A)
    assert np.abs(K.T @ K - Ainv).max() <= 2e-6 * np.abs(Ainv).max()
