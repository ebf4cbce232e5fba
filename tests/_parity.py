"""Frame parity checks shared by the GPU tests (north-star tolerances).

* positions: max |x_gpu - x_oracle| <= 1e-5 x bbox diagonal after every frame;
* contact set and stick/slip: the frame-end classification (reading A21: active <=> lambda_n > 0,
  stick <=> |ydot_f| <= r_f (mu lambda_n - |lambda_f|), P:L292-298 / P:L1650) identical for every
  unilateral contact outside the exclusion band, i.e. unless the ORACLE's values lie closer to a
  switching surface than the position tolerance can resolve (classify_with_band);
* applied impulse: the per-vertex J^T Theta lambda of the last L-G iteration (unique even where
  the rows of D are dependent and lambda is not, reading A31).
"""
import math

import numpy as np

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


def assert_impulse_parity(o, lam_g, theta_g, lam_o, theta_o, rel=1e-4):
    """Per-vertex J^T Theta lambda of the last L-G iteration, GPU vs oracle (theta_g as returned
    by the sim_debug_contact_state hook, per-contact triples): max over vertices
    and components within `rel` of the largest per-vertex impulse.  (The impulse enters
    x^{k+1} = A^-1 (b + h^2 J^T Theta lambda); a 1e-4 relative impulse error moves x by
    well under the 1e-5 bbox position tolerance on the scenes tested.)"""
    fg = applied_impulse(o, np.asarray(lam_g, float), rows_from_triples(o, theta_g))
    fo = applied_impulse(o, np.asarray(lam_o, float), np.asarray(theta_o, float))
    scale = np.abs(fo).max()
    err = np.abs(fg - fo).max()
    assert err <= rel * max(scale, 1e-300), (err, scale, err / max(scale, 1e-300))
    return err / max(scale, 1e-300)


def assert_frame_parity(o, x, v, xg, xo, tol, what="", **frame_kw):
    """Plain north-star position bound: max |x_gpu - x_oracle| <= tol (1e-5 x bbox diagonal)."""
    err = float(np.abs(xg - xo).max())
    assert err <= tol, (what, err, tol, err / tol)
    return err
