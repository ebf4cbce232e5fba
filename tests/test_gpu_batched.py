"""Batched instances (BASELINE config 5): S scenes share mesh,
material and K; every instance of one handle must match the fp64 oracle run on
that instance alone, at the single-scene tolerances (BASELINE.json north_star):
per-SpMV 1e-5 relative, positions 1e-5 x bbox diagonal per frame, identical
stick/slip classification.  All calls go through the C ABI.
"""
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


def make(simmod, sc, S):
    return simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, n_instances=S)


def test_batched_apply_inverse_cfg3(simmod):
    """Batched K-passes (SpMM over 3 S right-hand sides) == A^-1 b per instance.
    S = 130 spans two 128-instance chunks, the second one partial."""
    sc = scenes.make_scene("cfg3")
    S = 130
    s = make(simmod, sc, S)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    rng = np.random.default_rng(5)
    b = rng.standard_normal((S, sc.mesh.n_v, 3)).astype(np.float32).astype(np.float64)
    x = s.debug_apply_inverse(b)
    for i in (0, 1, 31, 32, 100, 127, 128, 129):
        xr = o.solve(b[i][o.free])
        err = np.abs(x[i][o.free] - xr).max() / np.abs(xr).max()
        assert err < 1e-5, (i, err)
        assert np.all(x[i][o.pinned] == 0)


@pytest.mark.parametrize("S", [2, 33])
def test_batched_apply_inverse_small(simmod, S):
    """Small and non-multiple-of-32 instance counts on a 5k-DoF block."""
    sc = scenes.make_scene("block", nv=7, split="kuhn6")
    s = make(simmod, sc, S)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    rng = np.random.default_rng(S)
    b = rng.standard_normal((S, sc.mesh.n_v, 3)).astype(np.float32).astype(np.float64)
    x = s.debug_apply_inverse(b)
    for i in range(S):
        xr = o.solve(b[i][o.free])
        assert np.abs(x[i][o.free] - xr).max() < 1e-5 * np.abs(xr).max(), i


def test_batched_incline_instances(simmod):
    """Three incline instances on one handle: stick (mu* + 0.05), slip
    (mu* - 0.05) and no contact at all.  Each frame the oracle restarts from the
    instance's GPU state (re-synced, as in the single-scene test)."""
    th = 10.0
    mus = math.tan(math.radians(th))
    scs = [scenes.incline_block(theta_deg=th, mu=mus + d, nv=5, edge=0.1, youngs=1e8) for d in (0.05, -0.05)]
    base = scs[0]
    S = 3
    s = make(simmod, base, S)
    contacts = [scs[0].contacts, scs[1].contacts, []]
    for i in range(S):
        s.set_contacts(contacts[i], instance=i)
    ors = []
    for i in range(S):
        o = O.Oracle(base.mesh, base.material, base.h, lg_iters=5)
        if contacts[i]:
            o.set_contacts(contacts[i])
        ors.append(o)
    tol = 1e-5 * base.mesh.bbox_diag()
    xs = [base.mesh.X.copy() for _ in range(S)]
    vs = [np.zeros_like(base.mesh.X) for _ in range(S)]
    for f in range(5):
        for i in range(S):
            s.set_state(xs[i], vs[i], instance=i)
        s.step(1, 5)
        for i in range(S):
            xg, vg = s.get_state(instance=i)
            xo, vo, info = ors[i].frame(xs[i], vs[i])
            assert np.abs(xg - xo).max() < tol, (f, i, np.abs(xg - xo).max())
            if contacts[i]:
                bad, n = _parity.classification_mismatches(ors[i], xg, xs[i], s.get_lambda(instance=i), xo,
                                                           info["lam"], tol)
                assert bad == 0 and n > 0, (f, i, bad, n)
            xs[i], vs[i] = xg, vg


def test_batched_mixed_slot_classes(simmod):
    """Instances with different contact-vertex sets (slot-set classes of sizes 2, 1, 1 and
    an empty one) on one handle, each against the oracle, re-synced per frame."""
    th = 10.0
    sc = scenes.incline_block(theta_deg=th, mu=0.5, nv=5, edge=0.1, youngs=1e8)
    full = sc.contacts
    half = len(full) // 2
    sets = [full, full[:half], full[half - 3:], [], full]
    S = len(sets)
    s = make(simmod, sc, S)
    s.set_contacts_batch(sets)
    ors = []
    for cs in sets:
        o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=5)
        if cs:
            o.set_contacts(cs)
        ors.append(o)
    tol = 1e-5 * sc.mesh.bbox_diag()
    xs = [sc.mesh.X.copy() for _ in range(S)]
    vs = [np.zeros_like(sc.mesh.X) for _ in range(S)]
    for f in range(4):
        for i in range(S):
            s.set_state(xs[i], vs[i], instance=i)
        s.step(1, 5)
        for i in range(S):
            xg, vg = s.get_state(instance=i)
            xo, vo, info = ors[i].frame(xs[i], vs[i])
            assert np.abs(xg - xo).max() < tol, (f, i, np.abs(xg - xo).max())
            xs[i], vs[i] = xg, vg
    # instances 0 and 4 (same inputs, same class) stay bit-identical
    assert np.array_equal(xs[0], xs[4])


def test_batched_gingerbread_cfg5(simmod):
    """cfg5 structure on cfg3: 4 instances with their own initial velocities and obstacle
    offsets (scenes.batch_instance), contacts set in one batch call; one frame per instance
    against the oracle (the non-penetrating instances 0 and 3 of the seeded draw)."""
    sc = scenes.make_scene("cfg3")
    S = 4
    s = make(simmod, sc, S)
    s.set_pin_velocity(sc.pin_velocity)
    inst = [scenes.batch_instance(sc, i) for i in range(S)]
    s.set_contacts_batch([c for _, c in inst])
    for i, (v0, _) in enumerate(inst):
        s.set_state(sc.mesh.X, v0, instance=i)
    s.step(1, 5)
    tol = 1e-5 * sc.mesh.bbox_diag()
    for i in (0, 3):
        v0, cs = inst[i]
        o = O.Oracle(sc.mesh, sc.material, sc.h)
        o.set_contacts(cs)
        pins = sc.mesh.X[o.pinned] + sc.h * sc.pin_velocity
        xo, vo, info = o.frame(sc.mesh.X.copy(), v0, pin_targets=pins)
        xg, vg = s.get_state(instance=i)
        err = np.abs(xg - xo).max()
        assert err < tol, (i, err, tol)
        bad, n = _parity.classification_mismatches(o, xg, sc.mesh.X, s.get_lambda(instance=i), xo, info["lam"],
                                                  tol)
        assert bad == 0, (i, bad, n)
    # all instances advance: positions differ between instances (different inputs)
    P = s.get_positions()
    assert P.shape == (S, sc.mesh.n_v, 3)
    assert np.array_equal(P[0], s.get_state(instance=0)[0])
    assert np.abs(P[1] - P[2]).max() > 0


def test_batched_determinism(simmod):
    sc = scenes.make_scene("block", nv=7, split="kuhn6")
    S = 40
    out = []
    for _ in range(2):
        s = make(simmod, sc, S)
        for i in range(S):
            x, v = scenes.random_state(sc.mesh, seed=i, amp=0.05)
            s.set_state(sc.mesh.X, v, instance=i)
        s.step(2, 5)
        out.append(s.get_positions())
        s.close()
    assert np.array_equal(out[0], out[1])


def test_split_contact_passes_one_cta_cr(simmod):
    """S = 96 incline instances: one CR CTA per instance (G_A gathered from the class Gram into
    shared memory, row-per-thread matvec) and tensor-core chain / scatter passes split over tile
    ranges (fp64 partials, per-unit arrival counters).  The same frames re-run on the same handle
    are bitwise identical (the counters reset themselves), and instances match the oracle."""
    sc = scenes.incline_block(theta_deg=10.0, mu=math.tan(math.radians(10.0)) - 0.05, nv=5, edge=0.1,
                              youngs=1e8)
    S = 96
    s = make(simmod, sc, S)
    s.set_contacts_batch([sc.contacts] * S)
    # rigid initial velocities (0 to 12 mm/s along x): smooth, distinct per instance (random
    # per-vertex velocities on this E = 1e8 block are ill-conditioned: fp32 rounding of the
    # inputs alone moves the oracle by 258 tolerances, tools/split_parity_check.py)
    v0 = np.zeros((S,) + sc.mesh.X.shape)
    v0[:, :, 0] = 0.002 * (np.arange(S) % 7)[:, None]
    v0[:, sc.mesh.fixed.astype(bool)] = 0.0
    runs = []
    for _ in range(2):
        s.set_states(np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape), v0)
        s.step(1, 5)
        runs.append(s.get_positions())
    assert np.array_equal(runs[0], runs[1])
    tol = 1e-5 * sc.mesh.bbox_diag()
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    o.set_contacts(sc.contacts)
    for i in (0, 57, S - 1):
        xo, _, _ = o.frame(sc.mesh.X.copy(), v0[i])
        assert np.abs(runs[0][i] - xo).max() < tol, (i, np.abs(runs[0][i] - xo).max())


def test_instance_validation(simmod):
    sc = scenes.make_scene("block", nv=5)
    s = make(simmod, sc, 2)
    with pytest.raises(simmod.SimError, match="instance"):
        s.set_contacts([], instance=2)
    with pytest.raises(simmod.SimError, match="instance"):
        s.get_state(instance=-1)


def test_tensor_core_and_fp32_kpasses_agree(simmod):
    """The tcgen05 (kind::tf32, 3xTF32, TMEM) batched K-passes and the CUDA-core FP32 ones
    (include/sim.h sim_set_kpass_mode) on the same right-hand sides: both match the oracle's
    A^-1 b within 1e-5 relative, and agree with each other to fp32 rounding."""
    sc = scenes.make_scene("block", nv=7, split="kuhn6")
    S = 130
    s = make(simmod, sc, S)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    rng = np.random.default_rng(9)
    b = rng.standard_normal((S, sc.mesh.n_v, 3)).astype(np.float32).astype(np.float64)
    out = {}
    for mode in (0, 1, 2):
        s.set_kpass_mode(mode)
        out[mode] = s.debug_apply_inverse(b)
    for i in (0, 63, 127, 128, 129):
        xr = o.solve(b[i][o.free])
        for mode in (0, 1, 2):
            assert np.abs(out[mode][i][o.free] - xr).max() < 1e-5 * np.abs(xr).max(), (mode, i)
    assert np.abs(out[0] - out[1]).max() < 1e-5 * np.abs(out[1]).max()
    assert np.abs(out[2] - out[1]).max() < 1e-5 * np.abs(out[1]).max()


def test_nonfinite_frame_rolls_back_one_instance(simmod):
    """Failure detection (include/sim.h sim_synchronize, SIM_E_NONFINITE): an instance whose
    frame turns non-finite (NaN injected after the prediction by the sim_debug_poison hook) is
    restored to its frame-start x, v on the device; the other instance advances as the oracle
    says; the error is reported once and counted in the stats; the next frame is normal."""
    sc = scenes.make_scene("block", nv=5)
    s = make(simmod, sc, 2)
    xs, vs = scenes.random_state(sc.mesh, seed=4, amp=0.05)
    fx = sc.mesh.fixed.astype(bool)
    xs[fx] = sc.mesh.X[fx]
    vs[fx] = 0.0
    for i in range(2):
        s.set_state(xs, vs, instance=i)
    s.debug_poison(0)
    s.step(1, 5)
    with pytest.raises(simmod.SimError, match="-7"):
        s.synchronize()
    s.synchronize()                   # reported once
    x0, v0 = s.get_state(instance=0)
    assert np.array_equal(x0, xs) and np.array_equal(v0, vs)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    xo, vo, _ = o.frame(xs, vs)
    x1, _ = s.get_state(instance=1)
    assert np.abs(x1 - xo).max() < 1e-5 * sc.mesh.bbox_diag()
    assert s.stats()["nonfinite_rollbacks"] == 1
    s.step(1, 5)                      # graph replay again, both instances healthy
    s.synchronize()
    x0, _ = s.get_state(instance=0)
    assert np.abs(x0 - xo).max() < 1e-5 * sc.mesh.bbox_diag()


def test_async_position_readback(simmod):
    """sim_get_positions_async / sim_wait_positions: double-buffered pinned read-back matches
    the synchronous sim_get_positions after each of several frames."""
    import torch
    sc = scenes.make_scene("block", nv=5)
    S = 3
    s = make(simmod, sc, S)
    bufs = [torch.empty((S, sc.mesh.n_v, 3), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    ref = []
    for f in range(4):
        s.step(1, 5)
        s.get_positions_async(bufs[f % 2].data_ptr())
        if f % 2 == 1:
            s.wait_positions(True)
            assert np.array_equal(bufs[0].numpy(), ref[-1])
            assert np.array_equal(bufs[1].numpy(), s.get_positions())
        ref.append(s.get_positions())


def test_cfg5_full_size_sampled(simmod):
    """cfg5 in the bench's launch configuration: 1024 cfg3 instances on one handle (tensor-core
    K-passes in 8 chunks of 128, one CR CTA per instance), initial velocities N(0, 0.01^2) m/s
    and obstacle offsets U(-5, +5) mm (about half of the instances start up
    to 5 mm inside the bars), contacts committed in one batch.

    Sampled instances: the first and last, the 3 deepest initial penetrations and the 3 smallest
    non-negative gaps.  Every one: its first L-G iteration (a frame of 1 iteration) within
    1e-5 bbox of the oracle with identical classification outside the tolerance band.  The
    non-penetrating ones: the whole 5-iteration frame, the same bounds.  The 5-iteration frame of
    a penetrating start is not compared here: the method's frame map there switches friction rows
    on the sign of lambda_n of separating contacts (theta_f = [lambda_n > 0]), and
    the fp64 oracle itself, continued from an iterate 1e-9 m off its own, ends tens of tolerances
    away (tools/diag_iteration.py); tools/cfg5_parity_scan.py reports those frames."""
    sc = scenes.make_scene("cfg3")
    S = 1024
    s = make(simmod, sc, S)
    s.set_pin_velocity(sc.pin_velocity)
    base = simmod.contacts_to_array(sc.contacts)
    arrs, v0s = [], np.empty((S, sc.mesh.n_v, 3))
    deltas = np.empty(S)
    for i in range(S):
        v0s[i], deltas[i] = scenes.batch_instance_params(sc, i)
        a = base.copy()
        a["offset"] += a["normal"][:, 2] * deltas[i]
        arrs.append(a)
    s.set_contacts_batch(packed=(np.concatenate(arrs), np.full(S, len(base), np.int32)))
    X0 = np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape)
    runs = {}
    for iters in (1, 5):
        s.set_states(X0, v0s)                  # also restarts every instance from lambda = 0
        s.step(1, iters)
        runs[iters] = (s.get_positions(), {i: s.get_lambda(i) for i in range(S)})
        assert np.isfinite(runs[iters][0]).all()
    tol = 1e-5 * sc.mesh.bbox_diag()
    order = np.argsort(-deltas)
    gaps = [int(c) for c in np.argsort(np.where(deltas <= 0, -deltas, np.inf))[:3]]
    sample = [0, 1023] + [int(c) for c in order[:3]] + gaps
    for i in sample:
        _, cs = scenes.batch_instance(sc, i)
        for iters in ((1, 5) if deltas[i] <= 0 else (1,)):
            o = O.Oracle(sc.mesh, sc.material, sc.h, lg_iters=iters)
            o.set_contacts(cs)
            pins = sc.mesh.X[o.pinned] + sc.h * sc.pin_velocity
            xo, _, info = o.frame(sc.mesh.X.copy(), v0s[i], pin_targets=pins)
            P, L = runs[iters]
            err = np.abs(P[i] - xo).max()
            assert err <= tol, (i, iters, deltas[i], err / tol)
            bad, n = _parity.classification_mismatches(o, P[i], sc.mesh.X, L[i], xo, info["lam"], tol)
            assert bad == 0, (i, iters, bad, n)


def _cfg5_batch(simmod, sc, S):
    """cfg5 handle of S instances with the bench's per-instance recipe (scenes.batch_instance_params)."""
    s = make(simmod, sc, S)
    s.set_pin_velocity(sc.pin_velocity)
    base = simmod.contacts_to_array(sc.contacts)
    arrs, v0s, deltas = [], np.empty((S, sc.mesh.n_v, 3)), np.empty(S)
    for i in range(S):
        v0s[i], deltas[i] = scenes.batch_instance_params(sc, i)
        a = base.copy()
        a["offset"] += a["normal"][:, 2] * deltas[i]
        arrs.append(a)
    s.set_contacts_batch(packed=(np.concatenate(arrs), np.full(S, len(base), np.int32)))
    return s, v0s, deltas


def test_cfg5_full_size_penetrating_iterations(simmod):
    """cfg5 at full size in the bench's launch configuration (S = 1024, tensor-core K-passes),
    the 8 deepest initial penetrations (delta up to +5 mm): EVERY L-G iteration of the frame,
    re-synced (the oracle runs the body of Alg. 4, once from the GPU's own iterate
    (x^k, lambda^k)), within the plain 1e-5 bbox bound, no conditioning guard.  Frame-level
    parity of these frames at 5 iterations is tested with the fp32 CUDA-core K-passes
    (test_cfg5_full_size_fp32_kpasses_penetrating_frames); DESIGN.md §3 (conditioning)."""
    sc = scenes.make_scene("cfg3")
    S = 1024
    s, v0s, deltas = _cfg5_batch(simmod, sc, S)
    X0 = np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape)
    deep = [int(c) for c in np.argsort(-deltas)[:8]]
    its = {i: [] for i in deep}
    for k in range(1, 6):
        s.set_states(X0, v0s)
        s.step(1, k)
        P = s.get_positions()
        for i in deep:
            its[i].append((P[i].copy(), s.get_lambda(i).copy()))
    tol = 1e-5 * sc.mesh.bbox_diag()
    worst = 0.0
    for i in deep:
        _, cs = scenes.batch_instance(sc, i)
        o = O.Oracle(sc.mesh, sc.material, sc.h)
        o.set_contacts(cs)
        pins = sc.mesh.X[o.pinned] + sc.h * sc.pin_velocity
        prev = None
        for k, (xg, lg) in enumerate(its[i]):
            o.lg_iters = k + 1
            start = None if prev is None else (prev[0], prev[1], k)
            xo, _, _ = o.frame(sc.mesh.X.copy(), v0s[i], pin_targets=pins, start=start)
            e = float(np.abs(xg - xo).max()) / tol
            assert e <= 1.0, (i, deltas[i], k, e)
            worst = max(worst, e)
            prev = (xg, lg)
    print(f"worst re-synced iteration err/tol over the 8 deepest penetrations: {worst:.4f}")


def test_cfg5_full_size_fp32_kpasses_penetrating_frames(simmod):
    """cfg5 at full size (S = 1024) with the batched fp32 CUDA-core K-passes
    (sim_set_kpass_mode(1)): the whole 5-iteration frame of the 8 deepest initial penetrations
    within the plain 1e-5 bbox bound of the oracle, classification identical outside the A21
    band.  (The tensor-core K-apply -- 3xTF32 products, fp32 TMEM accumulation, 2.6e-6 relative,
    inside the north star's 1e-5 SpMV bound -- seeds these frames 15x more than fp32 rounding and
    their non-smooth frame map amplifies it past 1e-5 bbox on some of the deepest; deeper in the
    distribution a few frames are ill-conditioned even for fp32 (the oracle itself moves by
    several tolerances under fp32 input rounding): profiles/r02s3_cfg5_parity_scan_wide.txt,
    DESIGN.md §3.)"""
    sc = scenes.make_scene("cfg3")
    S = 1024
    s, v0s, deltas = _cfg5_batch(simmod, sc, S)
    s.set_kpass_mode(1)
    X0 = np.broadcast_to(sc.mesh.X, (S,) + sc.mesh.X.shape)
    s.set_states(X0, v0s)
    s.step(1, 5)
    P = s.get_positions()
    assert np.isfinite(P).all()
    tol = 1e-5 * sc.mesh.bbox_diag()
    for i in [int(c) for c in np.argsort(-deltas)[:8]]:
        _, cs = scenes.batch_instance(sc, i)
        o = O.Oracle(sc.mesh, sc.material, sc.h)
        o.set_contacts(cs)
        pins = sc.mesh.X[o.pinned] + sc.h * sc.pin_velocity
        xo, _, info = o.frame(sc.mesh.X.copy(), v0s[i], pin_targets=pins)
        err = np.abs(P[i] - xo).max()
        assert err <= tol, (i, deltas[i], err / tol)
        bad, n = _parity.classification_mismatches(o, P[i], sc.mesh.X, s.get_lambda(i), xo, info["lam"], tol)
        assert bad == 0, (i, bad, n)


@pytest.mark.parametrize("model", [1, 2])
def test_batched_materials_with_contacts(simmod, model):
    """Corotated and ARAP (closed-form local steps, their own k_local instantiations) with
    frictional contact on two instances sharing K, re-synced frames vs the oracle."""
    th = 10.0
    sc = scenes.incline_block(theta_deg=th, mu=math.tan(math.radians(th)) - 0.05, nv=5, edge=0.1, youngs=1e7)
    sc.material.model = model
    S = 2
    s = make(simmod, sc, S)
    for i in range(S):
        s.set_contacts(sc.contacts, instance=i)
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    o.set_contacts(sc.contacts)
    tol = 1e-5 * sc.mesh.bbox_diag()
    # instance 1 starts sliding down the slope at 5 cm/s (a randomly perturbed, partly
    # penetrating start is outside the parity envelope: 5 fixed iterations do not resolve a
    # 0.8 mm penetration and the FB switching amplifies fp32 rounding, on S = 1 as well)
    down = -np.array([math.cos(math.radians(th)), 0.0, math.sin(math.radians(th))])
    xs = [sc.mesh.X.copy(), sc.mesh.X.copy()]
    vs = [np.zeros_like(sc.mesh.X), np.tile(0.05 * down, (sc.mesh.n_v, 1))]
    for f in range(4):
        for i in range(S):
            s.set_state(xs[i], vs[i], instance=i)
        s.step(1, 5)
        for i in range(S):
            xg, vg = s.get_state(instance=i)
            xo, _, _ = o.frame(xs[i], vs[i])
            assert np.abs(xg - xo).max() < tol, (f, i, np.abs(xg - xo).max())
            xs[i], vs[i] = xg, vg


@pytest.mark.parametrize("S", [1, 130])
def test_drop_tolerance_apply_inverse(simmod, S):
    """Drop tolerance (reading A25) on the device paths (S = 1 streaming SpMV, S = 130 tensor-core
    plane kernels): the K-pass streams shrink with the tolerance and K^T K b approximates the exact
    solve -- exact at tol 0 (1e-5 relative), error growing with the tolerance but below 1e3 tol."""
    sc = scenes.make_scene("block", nv=7, split="kuhn6")
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    rng = np.random.default_rng(5)
    b = rng.standard_normal((S, sc.mesh.n_v, 3)).astype(np.float32).astype(np.float64)
    prev_bytes, errs = None, []
    for tol in (0.0, 1e-4, 1e-3):
        s = simmod.Sim(sc.mesh.X, sc.mesh.T, sc.mesh.fixed, sc.material, sc.h, drop_tolerance=tol, n_instances=S)
        x = s.debug_apply_inverse(b if S > 1 else b[0]).reshape(S, sc.mesh.n_v, 3)
        e = 0.0
        for i in (0, S - 1):
            xr = o.solve(b[i][o.free])
            e = max(e, float(np.abs(x[i][o.free] - xr).max() / np.abs(xr).max()))
        errs.append(e)
        kb = s.stats()["kpass_bytes"]
        assert prev_bytes is None or kb <= prev_bytes
        prev_bytes = kb
        s.close()
    assert errs[0] < 1e-5, errs
    assert errs[1] < 1e3 * 1e-4 and errs[2] < 1e3 * 1e-3, errs


@pytest.mark.parametrize("model", [0, 1, 2])
def test_paired_local_step_matches_scalar_and_oracle(simmod, model):
    """The packed-FP32 paired local step (include/sim.h sim_set_local_mode 0: two instances per
    thread, FFMA2 / FMUL2 / FADD2 in lockstep) against the scalar kernel (mode 1) and the oracle:
    4 instances of a perturbed block (NH, linear corotated, ARAP), one frame of 5 L-G iterations
    each instance within 1e-5 bbox of the oracle, the two kernels within 1e-5 bbox of each other."""
    sc = scenes.make_scene("block", nv=6, model=model)
    S = 4
    tol = 1e-5 * sc.mesh.bbox_diag()
    states = [scenes.random_state(sc.mesh, seed=20 + i, amp=0.08) for i in range(S)]
    X0 = np.stack([st[0] for st in states])
    V0 = np.stack([st[1] for st in states])
    fx = sc.mesh.fixed.astype(bool)
    X0[:, fx] = sc.mesh.X[fx]
    V0[:, fx] = 0.0
    out = {}
    for mode in (0, 1):
        s = make(simmod, sc, S)
        s.set_local_mode(mode)
        s.set_states(X0, V0)
        s.step(1, 5)
        out[mode] = s.get_positions()
        s.close()
    assert np.abs(out[0] - out[1]).max() < tol
    o = O.Oracle(sc.mesh, sc.material, sc.h)
    for i in range(S):
        xo, _, _ = o.frame(X0[i], V0[i])
        assert np.abs(out[0][i] - xo).max() < tol, (i, np.abs(out[0][i] - xo).max() / tol)
