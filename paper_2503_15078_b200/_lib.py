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
    "sim_get_kernel_times", "sim_debug_contact_state", "sim_debug_cr_timeline", "sim_debug_pl_timeline", "sim_set_contacts_batch",
    "sim_get_positions", "sim_set_states", "sim_set_cr_mode", "sim_set_ncp", "sim_set_admm", "sim_set_kpass_mode", "sim_debug_poison", "sim_get_positions_async",
    "sim_wait_positions", "sim_detect_contacts", "sim_get_contacts",
    "sim_set_schur_reuse", "sim_set_lambda", "sim_set_pins", "sim_set_allocator", "sim_set_warm_start", "sim_set_persistent", "sim_set_local_mode", "sim_debug_contact_rho",
]
KERNEL_KINDS = ["predict", "contact_eval", "local", "gather", "kpass1", "chain_dot", "cr", "scatter", "kpass2", "active"]


class SimMesh(C.Structure):
    _fields_ = [("n_vertices", C.c_int32), ("n_tets", C.c_int32),
                ("rest_positions", C.POINTER(C.c_double)), ("tets", C.POINTER(C.c_int32)),
                ("fixed", C.POINTER(C.c_uint8)), ("n_instances", C.c_int32)]


class SimMaterial(C.Structure):
    _fields_ = [("model", C.c_int32), ("density", C.c_double), ("youngs", C.c_double),
                ("poisson", C.c_double), ("proj_stiffness", C.c_double),
                ("gravity", C.c_double * 3), ("cr_iterations", C.c_int32)]


class SimContact(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_verts", C.c_int32), ("verts", C.c_int32 * 4),
                ("weights", C.c_double * 4), ("normal", C.c_double * 3), ("tangent1", C.c_double * 3),
                ("tangent2", C.c_double * 3), ("offset", C.c_double),
                ("obstacle_velocity", C.c_double * 3), ("mu", C.c_double), ("compliance", C.c_double)]


# numpy twin of SimContact (same layout) for vectorised packing of large batches
CONTACT_DTYPE = np.dtype([("kind", "<i4"), ("n_verts", "<i4"), ("verts", "<i4", 4), ("weights", "<f8", 4),
                          ("normal", "<f8", 3), ("tangent1", "<f8", 3), ("tangent2", "<f8", 3),
                          ("offset", "<f8"), ("obstacle_velocity", "<f8", 3), ("mu", "<f8"),
                          ("compliance", "<f8")])
assert CONTACT_DTYPE.itemsize == C.sizeof(SimContact)


def contacts_to_array(contacts):
    """Contact objects -> CONTACT_DTYPE array (argument marshalling only)."""
    a = np.zeros(len(contacts), CONTACT_DTYPE)
    for i, ct in enumerate(contacts):
        n = len(ct.verts)
        a[i]["kind"] = int(getattr(ct, "kind", 0))
        a[i]["n_verts"] = n
        a[i]["verts"][:n] = [int(v) for v in ct.verts]
        a[i]["weights"][:n] = [float(w) for w in ct.weights]
        a[i]["normal"] = ct.normal
        t1, t2 = getattr(ct, "tangent1", None), getattr(ct, "tangent2", None)
        if t1 is not None:
            a[i]["tangent1"] = t1
        if t2 is not None:
            a[i]["tangent2"] = t2
        a[i]["offset"] = float(ct.offset)
        a[i]["obstacle_velocity"] = np.asarray(getattr(ct, "obstacle_velocity", np.zeros(3)))
        a[i]["mu"] = float(getattr(ct, "mu", 0.0))
        a[i]["compliance"] = float(getattr(ct, "compliance", 0.0))
    return a


class SimObstacle(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("a", C.c_double * 3), ("b", C.c_double * 3),
                ("radius", C.c_double), ("mu", C.c_double), ("velocity", C.c_double * 3)]


OBSTACLE_PLANE, OBSTACLE_SPHERE, OBSTACLE_CAPSULE = 0, 1, 2


class SimStats(C.Structure):
    _fields_ = [("n_vertices", C.c_int64), ("n_free", C.c_int64), ("n_tets", C.c_int64),
                ("nnz_K", C.c_int64), ("nnz_L", C.c_int64), ("etree_height", C.c_int32),
                ("n_panels", C.c_int32), ("n_contacts", C.c_int32), ("n_contact_vertices", C.c_int32),
                ("frames_done", C.c_int64), ("last_cr_residual", C.c_double), ("max_abs_phi_n", C.c_double),
                ("n_active", C.c_int32), ("n_stick", C.c_int32), ("n_slip", C.c_int32),
                ("kernels_per_frame", C.c_int32), ("build_seconds", C.c_double),
                ("h2d_contact_bytes", C.c_int64), ("n_instances", C.c_int32),
                ("nonfinite_rollbacks", C.c_int64), ("gram_rows_computed", C.c_int64),
                ("gram_rows_reused", C.c_int64), ("build_phase_seconds", C.c_double * 5),
                ("max_cone_violation", C.c_double), ("max_penetration", C.c_double), ("instance", C.c_int32),
                ("kpass_bytes", C.c_int64), ("nnz_K_kept", C.c_int64)]


class SimError(RuntimeError):
    pass


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)
_allocator_refs = []


def use_torch_allocator(on=True):
    """Route the library's device allocations through PyTorch's caching allocator
    (sim_set_allocator) for handles created afterwards; on=False restores cudaMalloc."""
    if not on:
        _check(lib.sim_set_allocator(None, None, None))
        return
    import torch

    def _alloc(nbytes, ctx):
        try:
            return int(torch.cuda.caching_allocator_alloc(int(nbytes)))
        except Exception:
            return None

    def _free(ptr, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    fa, ff = ALLOC_FN(_alloc), FREE_FN(_free)
    _allocator_refs[:] = [fa, ff]   # keep the trampolines alive while the library may call them
    _check(lib.sim_set_allocator(C.cast(fa, C.c_void_p), C.cast(ff, C.c_void_p), None))


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
        "sim_set_contacts": [H, C.c_int32, C.POINTER(SimContact), C.c_int32],
        "sim_set_contacts_batch": [H, C.c_int32, C.c_int32, ip, C.POINTER(SimContact)],
        "sim_get_positions": [H, dp],
        "sim_set_states": [H, dp, dp],
        "sim_step": [H, C.c_int32, C.c_int32],
        "sim_synchronize": [H],
        "sim_set_pin_velocity": [H, dp],
        "sim_get_state": [H, C.c_int32, dp, dp],
        "sim_set_state": [H, C.c_int32, dp, dp],
        "sim_get_lambda": [H, C.c_int32, dp, C.c_int32, C.POINTER(C.c_int32)],
        "sim_set_lambda": [H, C.c_int32, dp, C.c_int32],
        "sim_get_stats": [H, C.c_int32, C.POINTER(SimStats)],
        "sim_set_pins": [H, C.c_int32, dp, C.c_int32],
        "sim_set_allocator": [C.c_void_p, C.c_void_p, C.c_void_p],
        "sim_set_stream": [H, C.c_void_p],
        "sim_debug_get_inverse": [H, ip, ip, C.POINTER(C.c_int64), fp],
        "sim_debug_apply_inverse": [H, dp, dp],
        "sim_debug_local": [H, dp, dp, fp, dp],
        "sim_debug_get_delassus": [H, C.c_int32, ip, fp, C.c_int32],
        "sim_set_profiling": [H, C.c_int],
        "sim_set_cr_mode": [H, C.c_int32],
        "sim_set_ncp": [H, C.c_int32, C.c_int32],
        "sim_set_admm": [H, C.c_int32],
        "sim_set_warm_start": [H, C.c_int32],
        "sim_set_persistent": [H, C.c_int32],
        "sim_set_local_mode": [H, C.c_int32],
        "sim_set_kpass_mode": [H, C.c_int32],
        "sim_debug_poison": [H, C.c_int32],
        "sim_get_positions_async": [H, C.c_void_p],
        "sim_wait_positions": [H, C.c_int32],
        "sim_set_schur_reuse": [H, C.c_int32],
        "sim_get_contacts": [H, C.c_int32, C.POINTER(SimContact), C.c_int32, C.POINTER(C.c_int32)],
        "sim_detect_contacts": [H, C.c_int32, C.POINTER(SimObstacle), C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                C.c_double, C.POINTER(C.c_int32)],
        "sim_get_kernel_times": [H, dp, C.c_int32],
        "sim_debug_contact_state": [H, C.c_int32, dp, dp, dp, dp, ip, dp],
        "sim_debug_contact_rho": [H, C.c_int32, dp],
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
    """n_instances scenes sharing one mesh + material + h (and K), bound to the current device."""

    def __init__(self, X, T, fixed, material, h, drop_tolerance=0.0, host_only=False, n_instances=1):
        X = np.ascontiguousarray(X, dtype=np.float64)
        T = np.ascontiguousarray(T, dtype=np.int32)
        fixed = np.ascontiguousarray(fixed if fixed is not None else np.zeros(X.shape[0]), dtype=np.uint8)
        self.n_v, self.n_t = X.shape[0], T.shape[0]
        self.n_instances = int(n_instances)
        self._keep = (X, T, fixed)
        m = SimMesh(self.n_v, self.n_t, _dptr(X), T.ctypes.data_as(C.POINTER(C.c_int32)),
                    fixed.ctypes.data_as(C.POINTER(C.c_uint8)), self.n_instances)
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
        self._nc = [0] * self.n_instances
        self._contacts = [None] * self.n_instances

    @property
    def nc(self):
        return self._nc[0]

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

    def set_contacts(self, contacts=None, packed=None, instance=0):
        arr, n = packed if packed is not None else self.pack_contacts(contacts)
        _check(lib.sim_set_contacts(self._h, int(instance), arr, n))
        self._nc[instance] = n
        self._contacts[instance] = list(contacts) if contacts is not None else None

    def pack_contacts_batch(self, per_instance):
        """per_instance: list (one entry per instance) of contact lists -> packed batch."""
        counts = np.array([len(c) for c in per_instance], np.int32)
        arr = (SimContact * max(1, int(counts.sum())))()
        i = 0
        for cl in per_instance:
            for ct in cl:
                arr[i] = self._contact_struct(ct)
                i += 1
        return arr, counts

    def set_contacts_batch(self, per_instance=None, packed=None, first=0):
        """per_instance: list of contact lists, or packed = (contacts, counts) where contacts
        is a ctypes SimContact array or a CONTACT_DTYPE numpy array (concatenated)."""
        arr, counts = packed if packed is not None else self.pack_contacts_batch(per_instance)
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        if isinstance(arr, np.ndarray):
            assert arr.dtype == CONTACT_DTYPE and arr.flags.c_contiguous
            arr = arr.ctypes.data_as(C.POINTER(SimContact))
        _check(lib.sim_set_contacts_batch(self._h, int(first), len(counts),
                                          counts.ctypes.data_as(C.POINTER(C.c_int32)), arr))
        for k, n in enumerate(counts.tolist()):
            self._nc[first + k] = n
            self._contacts[first + k] = list(per_instance[k]) if per_instance is not None else None

    def step(self, frames=1, iterations=5):
        _check(lib.sim_step(self._h, int(frames), int(iterations)))

    def synchronize(self):
        _check(lib.sim_synchronize(self._h))

    def set_pin_velocity(self, v):
        a = np.ascontiguousarray(v, dtype=np.float64)
        _check(lib.sim_set_pin_velocity(self._h, _dptr(a)))

    def set_pins(self, targets, instance=0):
        """Positions the pinned vertices (ascending original index) take at the end of the next
        frame, [n_pinned][3] (sim_set_pins)."""
        a = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
        _check(lib.sim_set_pins(self._h, int(instance), _dptr(a), int(a.shape[0])))

    def get_state(self, instance=0):
        x = np.empty((self.n_v, 3))
        v = np.empty((self.n_v, 3))
        _check(lib.sim_get_state(self._h, int(instance), _dptr(x), _dptr(v)))
        return x, v

    def _f64(self, a, count, name):
        """Contiguous float64 copy of a, checked to hold exactly `count` values (the C side trusts sizes)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.size != count:
            raise ValueError(f"{name} must hold {count} values, got shape {a.shape}")
        return a

    def set_state(self, x, v, instance=0):
        x = self._f64(x, 3 * self.n_v, "x")
        v = self._f64(v, 3 * self.n_v, "v")
        _check(lib.sim_set_state(self._h, int(instance), _dptr(x), _dptr(v)))

    def set_states(self, x=None, v=None):
        """States of all instances, [n_instances][n_vertices][3] each (None = keep)."""
        n = 3 * self.n_v * self.n_instances
        xa = None if x is None else self._f64(x, n, "x")
        va = None if v is None else self._f64(v, n, "v")
        _check(lib.sim_set_states(self._h, None if xa is None else _dptr(xa), None if va is None else _dptr(va)))

    def get_positions(self, out=None):
        """Positions of all instances, [n_instances][n_vertices][3]."""
        if out is None:
            out = np.empty((self.n_instances, self.n_v, 3))
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != 3 * self.n_v * self.n_instances:
            raise ValueError("out must be a C-contiguous float64 array of n_instances x n_vertices x 3")
        _check(lib.sim_get_positions(self._h, _dptr(out)))
        return out

    def get_positions_async(self, out_ptr: int):
        """Enqueue the read-back of all positions into caller memory at address out_ptr
        ([n_instances][n_vertices][3] float64; pinned for overlap), sim_get_positions_async."""
        _check(lib.sim_get_positions_async(self._h, C.c_void_p(int(out_ptr))))

    def wait_positions(self, block_host: bool = True):
        _check(lib.sim_wait_positions(self._h, 1 if block_host else 0))

    def detect_contacts(self, obstacles, candidates, margin, instance=0):
        """GPU proximity query (sim_detect_contacts).  obstacles: list of dicts with kind
        (0 plane, 1 sphere, 2 capsule), a, b, radius, mu, velocity; candidates: original
        vertex ids.  Replaces the instance's contact set; returns the contact count."""
        arr = (SimObstacle * max(1, len(obstacles)))()
        for i, o in enumerate(obstacles):
            arr[i].kind = int(o["kind"])
            for k in range(3):
                arr[i].a[k] = float(o.get("a", (0, 0, 0))[k])
                arr[i].b[k] = float(o.get("b", (0, 0, 0))[k])
                arr[i].velocity[k] = float(o.get("velocity", (0, 0, 0))[k])
            arr[i].radius = float(o.get("radius", 0.0))
            arr[i].mu = float(o.get("mu", 0.0))
        cand = np.ascontiguousarray(candidates, dtype=np.int32)
        nf = C.c_int32(0)
        _check(lib.sim_detect_contacts(self._h, int(instance), arr, len(obstacles),
                                       cand.ctypes.data_as(C.POINTER(C.c_int32)), int(cand.size), float(margin),
                                       C.byref(nf)))
        self._nc[instance] = nf.value
        self._contacts[instance] = None
        return nf.value

    def get_contacts(self, instance=0):
        """The stored contact set of an instance as a CONTACT_DTYPE array (sim_get_contacts)."""
        n = C.c_int32(0)
        _check(lib.sim_get_contacts(self._h, int(instance), None, 0, C.byref(n)))
        arr = np.zeros(max(1, n.value), CONTACT_DTYPE)
        _check(lib.sim_get_contacts(self._h, int(instance), arr.ctypes.data_as(C.POINTER(SimContact)),
                                    int(arr.size), C.byref(n)))
        return arr[:n.value]

    def get_lambda(self, instance=0):
        """Multipliers the next frame of `instance` starts from (sim_get_lambda)."""
        n = C.c_int32(0)
        _check(lib.sim_get_lambda(self._h, int(instance), None, 0, C.byref(n)))
        out = np.empty(max(1, n.value))
        _check(lib.sim_get_lambda(self._h, int(instance), _dptr(out), out.size, C.byref(n)))
        return out[:n.value]

    def set_lambda(self, lam, instance=0):
        """Multipliers the next frame of `instance` starts from (sim_set_lambda)."""
        a = np.ascontiguousarray(lam, dtype=np.float64).reshape(-1)
        _check(lib.sim_set_lambda(self._h, int(instance), _dptr(a) if a.size else None, int(a.size)))

    def stats(self, instance=-1):
        """sim_get_stats: instance -1 = the whole handle, else that instance's contact fields."""
        s = SimStats()
        _check(lib.sim_get_stats(self._h, int(instance), C.byref(s)))
        out = {k: getattr(s, k) for k, _ in SimStats._fields_}
        out["build_phase_seconds"] = list(s.build_phase_seconds)
        return out

    def set_cr_mode(self, mode: int):
        """0 automatic, 1 cluster CR, 2 grid CR (include/sim.h sim_set_cr_mode)."""
        _check(lib.sim_set_cr_mode(self._h, int(mode)))

    def set_ncp(self, ncp: int = 0, precond: int = 0):
        """NCP function 0 FB / 1 min-map; preconditioner 0 Delassus / 1 mass inverse (sim_set_ncp)."""
        _check(lib.sim_set_ncp(self._h, int(ncp), int(precond)))

    def set_admm(self, on: bool = True):
        """ADMM-PD local-global variant (sim_set_admm)."""
        _check(lib.sim_set_admm(self._h, 1 if on else 0))

    def set_warm_start(self, on: bool = True):
        """Frame start (sim_set_warm_start): False x^0 = s, lambda^0 = 0 (readings A9/A10);
        True x^0 = x_t + h v_t, lambda carried from the previous frame (A9w/A10w)."""
        _check(lib.sim_set_warm_start(self._h, 1 if on else 0))

    def set_local_mode(self, mode: int):
        """Local step with several instances (sim_set_local_mode): 0 packed-FP32 instance pairs, 1 scalar."""
        _check(lib.sim_set_local_mode(self._h, int(mode)))

    def set_persistent(self, mode: int):
        """Small-scene driver (sim_set_persistent): 0 auto (one persistent kernel per sim_step for
        small contact-free single-instance scenes), 1 always the per-frame CUDA graph."""
        _check(lib.sim_set_persistent(self._h, int(mode)))

    def set_kpass_mode(self, mode: int):
        """Batched K-passes: 0 tensor cores (tcgen05), 1 CUDA-core FP32 (sim_set_kpass_mode)."""
        _check(lib.sim_set_kpass_mode(self._h, int(mode)))

    def debug_poison(self, instance=0):
        """Inject a NaN into the next frame of `instance` (sim_debug_poison)."""
        _check(lib.sim_debug_poison(self._h, int(instance)))

    def set_schur_reuse(self, on: bool = True):
        """Delassus Gram reuse across contact commits (sim_set_schur_reuse)."""
        _check(lib.sim_set_schur_reuse(self._h, 1 if on else 0))

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
        """b: [n_v][3] (single instance) or [n_instances][n_v][3]."""
        b = self._f64(b, 3 * self.n_v * self.n_instances, "b")
        x = np.empty(b.shape)
        _check(lib.sim_debug_apply_inverse(self._h, _dptr(b), _dptr(x)))
        return x

    def debug_local(self, x, s):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = np.ascontiguousarray(s, dtype=np.float64)
        P = np.empty((self.n_t, 3, 3), np.float32)
        r = np.empty((self.n_v, 3))
        _check(lib.sim_debug_local(self._h, _dptr(x), _dptr(s), P.ctypes.data_as(C.POINTER(C.c_float)), _dptr(r)))
        return P, r

    def _ns(self, instance):
        """Distinct contact vertices of an instance (from the stored set, sim_get_contacts)."""
        arr = self.get_contacts(instance)
        return len({int(v) for r in arr for v in r["verts"][:int(r["n_verts"])]})

    def debug_delassus(self, instance=0):
        ns = self._ns(instance)
        cv = np.empty(max(1, ns), np.int32)
        G = np.empty((max(1, ns), max(1, ns)), np.float32)
        _check(lib.sim_debug_get_delassus(self._h, int(instance), cv.ctypes.data_as(C.POINTER(C.c_int32)),
                                          G.ctypes.data_as(C.POINTER(C.c_float)), max(1, ns)))
        return cv[:ns], G[:ns, :ns]


def debug_contact_state(sim, instance=0):
    """Contact scratch of the last L-G iteration (see sim_debug_contact_state)."""
    nc, ns = sim._nc[instance], sim._ns(instance)
    th, cd, hv = np.empty(3 * nc), np.empty(3 * nc), np.empty(3 * nc)
    dxt = np.empty((max(1, ns), 3))
    sv = np.empty(max(1, ns), np.int32)
    djj = np.empty(max(1, nc))
    _check(lib.sim_debug_contact_state(sim._h, int(instance), _dptr(th), _dptr(cd), _dptr(hv), _dptr(dxt),
                                       sv.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(djj)))
    return {"theta": th, "cdiag": cd, "hvec": hv, "dxt": dxt[:ns], "slot_vertex": sv[:ns], "djj": djj[:nc]}


def debug_contact_rho(sim, instance=0):
    """Schur right-hand side of the last L-G iteration (sim_debug_contact_rho), per-contact triples."""
    out = np.empty(max(1, 3 * sim._nc[instance]))
    _check(lib.sim_debug_contact_rho(sim._h, int(instance), _dptr(out)))
    return out[:3 * sim._nc[instance]]


def debug_cr_timeline(sim):
    out = np.zeros(32)
    _check(lib.sim_debug_cr_timeline(sim._h, _dptr(out)))
    return out
