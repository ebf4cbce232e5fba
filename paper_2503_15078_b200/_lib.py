"""ctypes marshalling for include/sim.h (argument conversion only)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libsim.so")

MODEL_NEOHOOKEAN, MODEL_COROTATED, MODEL_ARAP = 0, 1, 2

EXPORTED_SYMBOLS = [
    "sim_create", "sim_create_host", "sim_build_sparse_inverse", "sim_set_contacts", "sim_step",
    "sim_synchronize", "sim_set_pin_velocity", "sim_get_state", "sim_set_state", "sim_get_lambda",
    "sim_get_stats", "sim_set_stream", "sim_destroy", "sim_last_error", "sim_debug_get_inverse",
    "sim_debug_apply_inverse", "sim_debug_local", "sim_debug_get_delassus", "sim_set_profiling",
    "sim_get_kernel_times", "sim_debug_contact_state", "sim_debug_cr_timeline",
]
KERNEL_KINDS = ["predict", "contact_eval", "local", "gather", "kpass1", "chain_dot", "cr", "scatter", "kpass2", "active"]


class SimMesh(C.Structure):
    _fields_ = [("n_vertices", C.c_int32), ("n_tets", C.c_int32),
                ("rest_positions", C.POINTER(C.c_double)), ("tets", C.POINTER(C.c_int32)),
                ("fixed", C.POINTER(C.c_uint8))]


class SimMaterial(C.Structure):
    _fields_ = [("model", C.c_int32), ("density", C.c_double), ("youngs", C.c_double),
                ("poisson", C.c_double), ("proj_stiffness", C.c_double),
                ("gravity", C.c_double * 3), ("cr_iterations", C.c_int32)]


class SimContact(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_verts", C.c_int32), ("verts", C.c_int32 * 4),
                ("weights", C.c_double * 4), ("normal", C.c_double * 3), ("tangent1", C.c_double * 3),
                ("tangent2", C.c_double * 3), ("offset", C.c_double),
                ("obstacle_velocity", C.c_double * 3), ("mu", C.c_double), ("compliance", C.c_double)]


class SimStats(C.Structure):
    _fields_ = [("n_vertices", C.c_int64), ("n_free", C.c_int64), ("n_tets", C.c_int64),
                ("nnz_K", C.c_int64), ("nnz_L", C.c_int64), ("etree_height", C.c_int32),
                ("n_panels", C.c_int32), ("n_contacts", C.c_int32), ("n_contact_vertices", C.c_int32),
                ("frames_done", C.c_int64), ("last_cr_residual", C.c_double), ("max_abs_phi_n", C.c_double),
                ("n_active", C.c_int32), ("n_stick", C.c_int32), ("n_slip", C.c_int32),
                ("kernels_per_frame", C.c_int32), ("build_seconds", C.c_double),
                ("h2d_contact_bytes", C.c_int64)]


class SimError(RuntimeError):
    pass


def _load():
    if not os.path.exists(lib_path):
        raise ImportError(f"{lib_path} not built; run paper_2503_15078_b200/build.py (no CPU fallback)")
    L = C.CDLL(lib_path)
    H = C.c_void_p
    dp, ip, fp = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_float)
    sig = {
        "sim_create": [C.POINTER(SimMesh), C.POINTER(SimMaterial), C.c_double, C.POINTER(H)],
        "sim_create_host": [C.POINTER(SimMesh), C.POINTER(SimMaterial), C.c_double, C.POINTER(H)],
        "sim_build_sparse_inverse": [H, C.c_double],
        "sim_set_contacts": [H, C.POINTER(SimContact), C.c_int32],
        "sim_step": [H, C.c_int32, C.c_int32],
        "sim_synchronize": [H],
        "sim_set_pin_velocity": [H, dp],
        "sim_get_state": [H, dp, dp],
        "sim_set_state": [H, dp, dp],
        "sim_get_lambda": [H, dp, C.c_int32],
        "sim_get_stats": [H, C.POINTER(SimStats)],
        "sim_set_stream": [H, C.c_void_p],
        "sim_debug_get_inverse": [H, ip, ip, C.POINTER(C.c_int64), fp],
        "sim_debug_apply_inverse": [H, dp, dp],
        "sim_debug_local": [H, dp, dp, fp, dp],
        "sim_debug_get_delassus": [H, ip, fp, C.c_int32],
        "sim_set_profiling": [H, C.c_int],
        "sim_get_kernel_times": [H, dp, C.c_int32],
        "sim_debug_contact_state": [H, dp, dp, dp, dp, ip, dp],
        "sim_debug_cr_timeline": [H, dp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.sim_destroy.argtypes = [H]
    L.sim_destroy.restype = None
    L.sim_last_error.argtypes = []
    L.sim_last_error.restype = C.c_char_p
    return L


lib = _load()


def _check(rc):
    if rc != 0:
        raise SimError(f"sim error {rc}: {lib.sim_last_error().decode()}")


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Sim:
    """One simulated object (mesh + material + h) bound to the current device."""

    def __init__(self, X, T, fixed, material, h, drop_tolerance=0.0, host_only=False):
        X = np.ascontiguousarray(X, dtype=np.float64)
        T = np.ascontiguousarray(T, dtype=np.int32)
        fixed = np.ascontiguousarray(fixed if fixed is not None else np.zeros(X.shape[0]), dtype=np.uint8)
        self.n_v, self.n_t = X.shape[0], T.shape[0]
        self._keep = (X, T, fixed)
        m = SimMesh(self.n_v, self.n_t, _dptr(X), T.ctypes.data_as(C.POINTER(C.c_int32)),
                    fixed.ctypes.data_as(C.POINTER(C.c_uint8)))
        g = (C.c_double * 3)(*[float(v) for v in material.gravity])
        mat = SimMaterial(int(material.model), float(material.density), float(material.youngs),
                          float(material.poisson), float(material.proj_stiffness), g,
                          int(material.cr_iterations))
        self._h = C.c_void_p()
        create = lib.sim_create_host if host_only else lib.sim_create
        _check(create(C.byref(m), C.byref(mat), float(h), C.byref(self._h)))
        self.host_only = host_only
        try:
            _check(lib.sim_build_sparse_inverse(self._h, float(drop_tolerance)))
        except Exception:
            self.close()
            raise
        self.nc = 0
        self._contacts = []

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.sim_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    @staticmethod
    def _contact_struct(ct):
        s = SimContact()
        s.kind = int(getattr(ct, "kind", 0))
        s.n_verts = len(ct.verts)
        for q, (v, w) in enumerate(zip(ct.verts, ct.weights)):
            s.verts[q] = int(v)
            s.weights[q] = float(w)
        for d in range(3):
            s.normal[d] = float(ct.normal[d])
            t1 = getattr(ct, "tangent1", None)
            t2 = getattr(ct, "tangent2", None)
            s.tangent1[d] = 0.0 if t1 is None else float(t1[d])
            s.tangent2[d] = 0.0 if t2 is None else float(t2[d])
            s.obstacle_velocity[d] = float(np.asarray(getattr(ct, "obstacle_velocity", np.zeros(3)))[d])
        s.offset = float(ct.offset)
        s.mu = float(getattr(ct, "mu", 0.0))
        s.compliance = float(getattr(ct, "compliance", 0.0))
        return s

    def pack_contacts(self, contacts):
        arr = (SimContact * max(1, len(contacts)))()
        for i, ct in enumerate(contacts):
            arr[i] = self._contact_struct(ct)
        return arr, len(contacts)

    def set_contacts(self, contacts=None, packed=None):
        arr, n = packed if packed is not None else self.pack_contacts(contacts)
        _check(lib.sim_set_contacts(self._h, arr, n))
        self.nc = n
        if contacts is not None:
            self._contacts = list(contacts)

    def step(self, frames=1, iterations=5):
        _check(lib.sim_step(self._h, int(frames), int(iterations)))

    def synchronize(self):
        _check(lib.sim_synchronize(self._h))

    def set_pin_velocity(self, v):
        a = np.ascontiguousarray(v, dtype=np.float64)
        _check(lib.sim_set_pin_velocity(self._h, _dptr(a)))

    def get_state(self):
        x = np.empty((self.n_v, 3))
        v = np.empty((self.n_v, 3))
        _check(lib.sim_get_state(self._h, _dptr(x), _dptr(v)))
        return x, v

    def set_state(self, x, v):
        x = np.ascontiguousarray(x, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        _check(lib.sim_set_state(self._h, _dptr(x), _dptr(v)))

    def get_lambda(self):
        cap = 3 * max(1, self.nc)
        out = np.empty(cap)
        _check(lib.sim_get_lambda(self._h, _dptr(out), cap))
        rows = sum(1 if getattr(c, "kind", 0) == 1 else 3 for c in self._contacts) if self._contacts else 3 * self.nc
        return out[:rows]

    def stats(self):
        s = SimStats()
        _check(lib.sim_get_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in SimStats._fields_}

    def set_profiling(self, on: bool):
        _check(lib.sim_set_profiling(self._h, 1 if on else 0))

    def kernel_times(self):
        out = np.zeros(len(KERNEL_KINDS))
        _check(lib.sim_get_kernel_times(self._h, _dptr(out), len(KERNEL_KINDS)))
        return dict(zip(KERNEL_KINDS, out.tolist()))

    def set_stream(self, stream_ptr: int):
        _check(lib.sim_set_stream(self._h, C.c_void_p(stream_ptr)))

    # ------------------------------------------------------------------ hooks
    def debug_inverse(self):
        st = self.stats()
        nf, nnz = int(st["n_free"]), int(st["nnz_K"])
        perm = np.empty(nf, np.int32)
        parent = np.empty(nf, np.int32)
        rowptr = np.empty(nf + 1, np.int64)
        vals = np.empty(nnz, np.float32)
        _check(lib.sim_debug_get_inverse(self._h, perm.ctypes.data_as(C.POINTER(C.c_int32)),
                                         parent.ctypes.data_as(C.POINTER(C.c_int32)),
                                         rowptr.ctypes.data_as(C.POINTER(C.c_int64)),
                                         vals.ctypes.data_as(C.POINTER(C.c_float))))
        return perm, parent, rowptr, vals

    def debug_apply_inverse(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty((self.n_v, 3))
        _check(lib.sim_debug_apply_inverse(self._h, _dptr(b), _dptr(x)))
        return x

    def debug_local(self, x, s):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = np.ascontiguousarray(s, dtype=np.float64)
        P = np.empty((self.n_t, 3, 3), np.float32)
        r = np.empty((self.n_v, 3))
        _check(lib.sim_debug_local(self._h, _dptr(x), _dptr(s), P.ctypes.data_as(C.POINTER(C.c_float)), _dptr(r)))
        return P, r

    def debug_delassus(self):
        ns = int(self.stats()["n_contact_vertices"])
        cv = np.empty(max(1, ns), np.int32)
        G = np.empty((max(1, ns), max(1, ns)), np.float32)
        _check(lib.sim_debug_get_delassus(self._h, cv.ctypes.data_as(C.POINTER(C.c_int32)),
                                          G.ctypes.data_as(C.POINTER(C.c_float)), max(1, ns)))
        return cv[:ns], G[:ns, :ns]


def debug_contact_state(sim):
    """Contact scratch of the last L-G iteration (see sim_debug_contact_state)."""
    st = sim.stats()
    nc, ns = int(st["n_contacts"]), int(st["n_contact_vertices"])
    th, cd, hv = np.empty(3 * nc), np.empty(3 * nc), np.empty(3 * nc)
    dxt = np.empty((max(1, ns), 3))
    sv = np.empty(max(1, ns), np.int32)
    djj = np.empty(max(1, nc))
    _check(lib.sim_debug_contact_state(sim._h, _dptr(th), _dptr(cd), _dptr(hv), _dptr(dxt),
                                       sv.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(djj)))
    return {"theta": th, "cdiag": cd, "hvec": hv, "dxt": dxt[:ns], "slot_vertex": sv[:ns], "djj": djj[:nc]}


def debug_cr_timeline(sim):
    out = np.zeros(32)
    _check(lib.sim_debug_cr_timeline(sim._h, _dptr(out)))
    return out
