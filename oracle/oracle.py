"""CPU oracle for the aligned-MSD / path-CV / floating-close-structure hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this module;
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may use it, and only as the checker / CPU baseline.

Two layers:

* A per-pair restatement of the reference geometry module
  (``/root/reference/pkg/src/metadyn_close/geometry.py``), function by function,
  each citing the reference line range it follows.  It is pinned against the
  golden vectors in ``tests/golden/`` that were produced by importing the
  reference itself (``tests/golden/make_golden.py``).
* A restatement of the parts that exist only as prose in the reference
  (``SPEC.md`` msd-engine + colvar modules, ``PAPER.md`` Eq. 2-6, Alg. 1-2):
  exact / approximate distances with gradients, the close-structure
  lifecycle, the property-map CV ``s`` and the builder-defined path-CV ``z``.
  Those are pinned by the SPEC's known-answer examples and by finite
  differences (``tests/test_oracle.py``); ``z`` is a non-goal of the
  reference (``SPEC.md:250``) and its parity is "unpinned" at the reference
  boundary.

A third, vectorised layer (``batch_*``) restates the same maths with numpy
batched LAPACK ``eigh`` so that parity tests can check thousands of pairs in
seconds; it is itself checked against the per-pair layer in the CPU tests.
"""

from __future__ import annotations

import math

import numpy as np

DEGENERACY_TOL = 1e-9  # geometry.py:22


class OracleError(Exception):
    pass


class InvalidStructure(OracleError):
    pass


class DegenerateFit(OracleError):
    pass


# --------------------------------------------------------------------------
# geometry.py restatement
# --------------------------------------------------------------------------

def normalise_weights(w, n):
    """geometry.py:49-61 — default 1/n, else validate and divide by the sum."""
    if w is None:
        return np.full(n, 1.0 / n)
    w = np.array(w, dtype=float)
    if w.shape != (n,):
        raise InvalidStructure("weights must have length n")
    if not np.all(np.isfinite(w)) or np.any(w < 0.0):
        raise InvalidStructure("weights must be finite and non-negative")
    total = w.sum()
    if total <= 0.0:
        raise InvalidStructure("weights sum to zero")
    return w / total


def validate_coords(coords):
    """geometry.py:35-42."""
    coords = np.array(coords, dtype=float)
    if coords.ndim != 2 or coords.shape[1] != 3:
        raise InvalidStructure("coords must be (n, 3)")
    if coords.shape[0] < 2:
        raise InvalidStructure("a structure needs at least 2 atoms")
    if not np.all(np.isfinite(coords)):
        raise InvalidStructure("coords contain non-finite values")
    return coords


def centroid(x, w_align):
    """geometry.py:67-69 — alignment-weighted centroid ``w' @ x``."""
    return w_align @ x


def center(x, w_align):
    """geometry.py:74-76 — ``x - centroid``."""
    return x - centroid(x, w_align)


def jacobi_eigh(mat, tol=1e-14, max_sweeps=60):
    """geometry.py:106-153 — cyclic Jacobi, ascending order, sign rule.

    Same rotation formula, same tolerance floor ``max(tol, 4e-16 |A|_F)``,
    same stable argsort and "largest-|component| positive" convention.
    """
    a = np.array(mat, dtype=float)
    n = a.shape[0]
    if a.shape != (n, n) or not np.allclose(a, a.T, atol=1e-12 * max(1.0, np.abs(a).max())):
        raise ValueError("jacobi_eigh expects a symmetric square matrix")
    v = np.eye(n)
    tol = max(tol, 4e-16 * np.linalg.norm(a))
    mask = ~np.eye(n, dtype=bool)
    for _ in range(max_sweeps):
        if math.sqrt(np.sum(a[mask] ** 2)) < tol:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                if apq == 0.0:
                    continue
                theta = (a[q, q] - a[p, p]) / (2.0 * apq)
                t = math.copysign(1.0, theta) / (abs(theta) + math.hypot(theta, 1.0))
                c = 1.0 / math.sqrt(t * t + 1.0)
                s = t * c
                cp, cq = a[:, p].copy(), a[:, q].copy()
                a[:, p], a[:, q] = c * cp - s * cq, s * cp + c * cq
                rp, rq = a[p, :].copy(), a[q, :].copy()
                a[p, :], a[q, :] = c * rp - s * rq, s * rp + c * rq
                a[p, q] = a[q, p] = 0.0
                vp, vq = v[:, p].copy(), v[:, q].copy()
                v[:, p], v[:, q] = c * vp - s * vq, s * vp + c * vq
    else:
        raise RuntimeError("Jacobi diagonalisation did not converge")
    order = np.argsort(np.diag(a), kind="stable")
    w = np.diag(a)[order]
    v = v[:, order]
    for j in range(n):
        i = int(np.argmax(np.abs(v[:, j])))
        if v[i, j] < 0.0:
            v[:, j] = -v[:, j]
    return w, v


def quat_to_rot(q):
    """geometry.py:156-164 — scalar-first unit quaternion to R."""
    q0, q1, q2, q3 = q
    return np.array([
        [q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2.0 * (q1 * q2 - q0 * q3), 2.0 * (q1 * q3 + q0 * q2)],
        [2.0 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2.0 * (q2 * q3 - q0 * q1)],
        [2.0 * (q1 * q3 - q0 * q2), 2.0 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3],
    ])


def rot_quat_jacobian(q):
    """geometry.py:167-177 — dR/dq_c, shape (4, 3, 3)."""
    q0, q1, q2, q3 = q
    return 2.0 * np.array([
        [[q0, -q3, q2], [q3, q0, -q1], [-q2, q1, q0]],
        [[q1, q2, q3], [q2, -q1, -q0], [q3, q0, -q1]],
        [[-q2, q1, q0], [q1, q2, q3], [-q0, q3, -q2]],
        [[-q3, -q0, q1], [q0, -q3, q2], [q1, q2, q3]],
    ])


def kearsley_matrix(x, a, w):
    """geometry.py:180-196 — 4x4 form from m = x - a, p = x + a."""
    m = x - a
    p = x + a
    wm = w[:, None] * m
    k = np.empty((4, 4))
    k[0, 0] = np.sum(wm * m)
    off = -np.sum(w[:, None] * np.cross(p, m), axis=0)
    k[0, 1:] = off
    k[1:, 0] = off
    k[1:, 1:] = wm.T @ m + np.eye(3) * np.sum(w * np.sum(p * p, axis=1)) - (w[:, None] * p).T @ p
    return k


def kearsley_matrix_grad(a, p, w):
    """geometry.py:199-224 — dK/dx_{k,alpha}, shape (n, 3, 4, 4)."""
    n = a.shape[0]
    m = p - 2.0 * a
    eye = np.eye(3)
    grad = np.zeros((n, 3, 4, 4))
    grad[:, :, 0, 0] = 2.0 * w[:, None] * m
    ax = np.zeros((n, 3, 3))
    ax[:, 0, 1] = -a[:, 2]
    ax[:, 0, 2] = a[:, 1]
    ax[:, 1, 0] = a[:, 2]
    ax[:, 1, 2] = -a[:, 0]
    ax[:, 2, 0] = -a[:, 1]
    ax[:, 2, 1] = a[:, 0]
    off = -2.0 * w[:, None, None] * ax.transpose(0, 2, 1)
    grad[:, :, 0, 1:] = off
    grad[:, :, 1:, 0] = off
    t1 = np.einsum("ab,kg->kabg", eye, a)
    block = -2.0 * (t1 + t1.transpose(0, 1, 3, 2)) + 2.0 * np.einsum("ka,bg->kabg", p, eye)
    grad[:, :, 1:, 1:] = w[:, None, None, None] * block
    return grad


def kearsley_fit(x, a, w, with_derivatives=False):
    """geometry.py:227-263.

    ``x`` (fitted) and ``a`` (reference) are centred (n,3) arrays, ``w`` the
    normalised displacement weights of ``x``.  Returns a dict with ``rot``,
    ``quat``, ``eigvals``, ``eigvecs`` and (optionally) ``rot_grad``.
    """
    if x.shape != a.shape:
        raise InvalidStructure("atom count mismatch")
    kmat = kearsley_matrix(x, a, w)
    eigvals, eigvecs = jacobi_eigh(kmat)
    quat = eigvecs[:, 0]
    rot = quat_to_rot(quat)
    rot_grad = None
    if with_derivatives:
        if eigvals[1] - eigvals[0] < DEGENERACY_TOL:
            raise DegenerateFit("eigenvalue gap below tolerance")
        dk = kearsley_matrix_grad(a, x + a, w)
        rest = eigvecs[:, 1:]
        coef = np.einsum("kaij,j->kai", dk, quat) @ rest
        coef /= (eigvals[0] - eigvals[1:])[None, None, :]
        dq = coef @ rest.T
        rot_grad = np.einsum("kac,cbg->kabg", dq, rot_quat_jacobian(quat))
    return {"rot": rot, "quat": quat, "eigvals": eigvals, "eigvecs": eigvecs, "rot_grad": rot_grad}


def rotation_derivative_check(x, a, w, h=1e-6):
    """geometry.py:266-285 — central differences of R, no re-centring."""
    fit = kearsley_fit(x, a, w, with_derivatives=True)
    worst = 0.0
    for k in range(x.shape[0]):
        for alpha in range(3):
            b = x.copy()
            b[k, alpha] += h
            rp = kearsley_fit(b, a, w)["rot"]
            b[k, alpha] -= 2.0 * h
            rm = kearsley_fit(b, a, w)["rot"]
            fd = (rp - rm) / (2.0 * h)
            worst = max(worst, float(np.abs(fd - fit["rot_grad"][k, alpha]).max()))
    return worst / max(1.0, float(np.abs(fit["rot_grad"]).max()))


# --------------------------------------------------------------------------
# msd-engine restatement (Eq. 3-6, Alg. 1-2)
# --------------------------------------------------------------------------

def _uncenter(g, w_align):
    """Chain rule through x_c = x - w'@x: g_raw_k = g_k - w'_k sum_j g_j."""
    return g - w_align[:, None] * g.sum(axis=0)[None, :]


def exact_distance(xc, ac, w, w_align, with_rot_term=True):
    """Eq. 3/4.

    D = sum_j w_j |x_j - R a_j|^2 with R = kearsley_fit(x, a).rot.  The
    gradient is w.r.t. the raw (uncentred) coordinates of x: 2 w d, plus the
    dR contraction term (zero at the optimum; kept here so the oracle states
    Eq. 4 literally), then the alignment-weight term of Eq. 4.
    """
    fit = kearsley_fit(xc, ac, w, with_derivatives=with_rot_term)
    rot = fit["rot"]
    d = xc - ac @ rot.T
    value = float(np.sum(w * np.sum(d * d, axis=1)))
    g = 2.0 * w[:, None] * d
    if with_rot_term:
        mmat = -2.0 * (w[:, None] * d).T @ ac  # dD/dR_{beta,gamma}
        g = g + np.einsum("bg,kabg->ka", mmat, fit["rot_grad"])
    return value, _uncenter(g, w_align), fit


def approx_distance(xc, ac, rot_ay, fit_xy, w, w_align):
    """Eq. 5/6.

    D~ = sum_j w_j |x_j - R_xy R_{a y} a_j|^2; gradient 2 w d~ plus the
    contraction of M = -2 sum_j w_j d~_j b_j^T (b = R_{ay} a) with
    dR_xy/dx (fit_xy must carry rot_grad), then the alignment-weight term.
    """
    b = ac @ rot_ay.T
    rxy = fit_xy["rot"]
    d = xc - b @ rxy.T
    value = float(np.sum(w * np.sum(d * d, axis=1)))
    mmat = -2.0 * (w[:, None] * d).T @ b
    g = 2.0 * w[:, None] * d + np.einsum("bg,kabg->ka", mmat, fit_xy["rot_grad"])
    return value, _uncenter(g, w_align)


# --------------------------------------------------------------------------
# colvar restatement (Eq. 2) + builder-defined z
# --------------------------------------------------------------------------

def property_map(dist, grads, q, lam):
    """Eq. 2 with the min-D shift.

    s = sum q_i e^{-lam D_i} / sum e^{-lam D_i};
    ds = -lam sum_i p_i (q_i - s) dD_i  (quotient rule).
    """
    dist = np.asarray(dist, dtype=float)
    if dist.size == 0:
        raise OracleError("empty active set")
    if not np.all(np.isfinite(dist)):
        raise OracleError("non-finite distances")
    q = np.asarray(q, dtype=float)
    e = np.exp(-lam * (dist - dist.min()))
    p = e / e.sum()
    s = float(np.dot(p, q))
    ds = None
    if grads is not None:
        c = -lam * p * (q - s)
        ds = np.einsum("i,ika->ka", c, grads)
    return s, ds


def path_z(dist, grads, lam):
    """Builder-defined path-CV z (Branduardi form).

    z = -(1/lam) ln sum_i e^{-lam D_i} = D_min - (1/lam) ln sum e^{-lam (D_i - D_min)};
    dz = sum_i p_i dD_i.
    """
    dist = np.asarray(dist, dtype=float)
    dmin = dist.min()
    e = np.exp(-lam * (dist - dmin))
    z = float(dmin - math.log(e.sum()) / lam)
    dz = None
    if grads is not None:
        p = e / e.sum()
        dz = np.einsum("i,ika->ka", p, grads)
    return z, dz


# --------------------------------------------------------------------------
# Drivers: exact path-CV (Alg. 1) and close-structure replay (Alg. 2)
# --------------------------------------------------------------------------

def path_cv_exact(frames, landmarks, lam, q=None, w=None, w_align=None, grad=True,
                  with_rot_term=True):
    """Alg. 1 without neighbour list: exact D_i for all i."""
    frames = np.asarray(frames, dtype=float)
    landmarks = np.asarray(landmarks, dtype=float)
    t_count, n, _ = frames.shape
    n_l = landmarks.shape[0]
    w = normalise_weights(w, n)
    wa = normalise_weights(w_align, n)
    q = np.arange(n_l, dtype=float) if q is None else np.asarray(q, dtype=float)
    lc = np.stack([center(a, wa) for a in landmarks])
    out = {"s": np.zeros(t_count), "z": np.zeros(t_count), "D": np.zeros((t_count, n_l))}
    if grad:
        out["ds"] = np.zeros((t_count, n, 3))
        out["dz"] = np.zeros((t_count, n, 3))
    for t in range(t_count):
        xc = center(frames[t], wa)
        dist = np.zeros(n_l)
        grads = np.zeros((n_l, n, 3)) if grad else None
        for i in range(n_l):
            if grad:
                dist[i], grads[i], _ = exact_distance(xc, lc[i], w, wa, with_rot_term=with_rot_term)
            else:
                dist[i] = kearsley_fit(xc, lc[i], w)["eigvals"][0]
        out["D"][t] = dist
        out["s"][t], ds = property_map(dist, grads, q, lam)
        out["z"][t], dz = path_z(dist, grads, lam)
        if grad:
            out["ds"][t], out["dz"][t] = ds, dz
    return out


def neighbour_update(distances, m):
    """SPEC neighbourlist maybe_update (SPEC.md: [MODULE] neighbourlist, OP
    maybe_update): indices of the m smallest distances, ties broken by the lower
    index, sorted ascending.  m > N -> configuration error."""
    d = np.asarray(distances, dtype=float)
    if not 1 <= m <= d.shape[-1]:
        raise ValueError("neighbour list size must satisfy 1 <= M <= N")
    order = np.lexsort((np.arange(d.shape[-1]), d))  # primary: distance, secondary: index
    return np.sort(order[:m])


def close_structure_replay(frames, landmarks, lam, eps, q=None, w=None, w_align=None,
                           grad=True, neighbours=None, nl_stride=1):
    """Alg. 2.

    Per frame: centre x; always one exact fit x<->y with derivatives (first
    frame: y := x, D(x,y) := 0); refresh if first frame or D(x,y) > eps
    (strict).  On refresh y <- x_c, the saved rotations R_{a_i y} are refit
    exactly and the exact distances are returned; otherwise the Eq. 5/6
    approximations are returned for every landmark.

    neighbours = M (optional): SPEC neighbourlist in close-structure mode -- at
    frames 0, nl_stride, 2 nl_stride, ... the list is updated from that frame's
    distances to ALL landmarks (approximated on non-refresh frames, exact on
    refresh frames); s, z and their gradients sum over the active set only
    (SPEC colvar "active set").
    """
    frames = np.asarray(frames, dtype=float)
    landmarks = np.asarray(landmarks, dtype=float)
    t_count, n, _ = frames.shape
    n_l = landmarks.shape[0]
    w = normalise_weights(w, n)
    wa = normalise_weights(w_align, n)
    q = np.arange(n_l, dtype=float) if q is None else np.asarray(q, dtype=float)
    lc = np.stack([center(a, wa) for a in landmarks])
    out = {
        "s": np.zeros(t_count), "z": np.zeros(t_count), "D": np.zeros((t_count, n_l)),
        "refresh": np.zeros(t_count, dtype=bool), "dxy": np.zeros(t_count),
    }
    if grad:
        out["ds"] = np.zeros((t_count, n, 3))
        out["dz"] = np.zeros((t_count, n, 3))
    y = None
    saved = None
    active = None
    counters = {"step_count": 0, "reassign_count": 0, "expensive_count": 0, "cheap_count": 0}
    for t in range(t_count):
        xc = center(frames[t], wa)
        counters["step_count"] += 1
        counters["expensive_count"] += 1
        if y is None:
            dxy = 0.0
            fit_xy = None
            refresh = True
        else:
            fit_xy = kearsley_fit(xc, y, w, with_derivatives=True)
            dxy = float(fit_xy["eigvals"][0])
            refresh = dxy > eps
        out["dxy"][t] = dxy
        out["refresh"][t] = refresh
        dist = np.zeros(n_l)
        grads = np.zeros((n_l, n, 3)) if grad else None
        if refresh:
            y = xc.copy()
            saved = np.zeros((n_l, 3, 3))
            counters["reassign_count"] += 1
            counters["expensive_count"] += n_l
            for i in range(n_l):
                if grad:
                    dist[i], grads[i], fit = exact_distance(xc, lc[i], w, wa)
                else:
                    fit = kearsley_fit(xc, lc[i], w)
                    dist[i] = fit["eigvals"][0]
                saved[i] = fit["rot"]
        else:
            counters["cheap_count"] += n_l
            for i in range(n_l):
                dist[i], g = approx_distance(xc, lc[i], saved[i], fit_xy, w, wa)
                if grad:
                    grads[i] = g
        out["D"][t] = dist
        if neighbours is not None:
            if t % nl_stride == 0:
                active = neighbour_update(dist, neighbours)
            out.setdefault("active", np.zeros((t_count, neighbours), dtype=np.int64))[t] = active
            da, ga_ = dist[active], (grads[active] if grad else None)
            out["s"][t], ds = property_map(da, ga_, q[active], lam)
            out["z"][t], dz = path_z(da, ga_, lam)
        else:
            out["s"][t], ds = property_map(dist, grads, q, lam)
            out["z"][t], dz = path_z(dist, grads, lam)
        if grad:
            out["ds"][t], out["dz"][t] = ds, dz
    out["counters"] = counters
    return out


# --------------------------------------------------------------------------
# Vectorised restatement (same maths, batched numpy eigh) for larger checks
# --------------------------------------------------------------------------

def _sign_fix(vecs):
    """geometry.py:149-152 on batched column eigenvectors (..., 4, 4)."""
    idx = np.argmax(np.abs(vecs), axis=-2)  # (..., 4)
    picked = np.take_along_axis(vecs, idx[..., None, :], axis=-2)[..., 0, :]
    sign = np.where(picked < 0.0, -1.0, 1.0)
    return vecs * sign[..., None, :]


def batch_kearsley_matrices(xc, ac, w):
    """Batched geometry.py:180-196 for xc (..., n, 3), ac (..., n, 3)."""
    m = xc - ac
    p = xc + ac
    wm = w[..., :, None] * m
    shape = np.broadcast_shapes(xc.shape, ac.shape)[:-2]
    k = np.empty(shape + (4, 4))
    k[..., 0, 0] = np.sum(wm * m, axis=(-1, -2))
    off = -np.sum(w[..., :, None] * np.cross(p, m), axis=-2)
    k[..., 0, 1:] = off
    k[..., 1:, 0] = off
    gp = np.sum(w * np.sum(p * p, axis=-1), axis=-1)
    k[..., 1:, 1:] = (np.einsum("...ja,...jb->...ab", wm, m)
                      + np.eye(3) * gp[..., None, None]
                      - np.einsum("...ja,...jb->...ab", w[..., :, None] * p, p))
    return k


def batch_fit(xc, ac, w):
    """Batched kearsley_fit (no derivatives): eigvals (...,4), quat (...,4), rot (...,3,3)."""
    k = batch_kearsley_matrices(xc, ac, w)
    vals, vecs = np.linalg.eigh(k)
    vecs = _sign_fix(vecs)
    quat = vecs[..., :, 0]
    q0, q1, q2, q3 = (quat[..., i] for i in range(4))
    rot = np.stack([
        np.stack([q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2)], -1),
        np.stack([2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1)], -1),
        np.stack([2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3], -1),
    ], -2)
    return vals, quat, rot, vecs


def batch_center(x, w_align):
    return x - np.einsum("j,...ja->...a", w_align, x)[..., None, :]


def batch_msd_matrix(frames, landmarks, w=None, w_align=None, block=64):
    """All-pairs exact MSD [T, L] (eigvals[0] of every frame/landmark fit)."""
    frames = np.asarray(frames, dtype=float)
    landmarks = np.asarray(landmarks, dtype=float)
    n = frames.shape[1]
    w = normalise_weights(w, n)
    wa = normalise_weights(w_align, n)
    fc = batch_center(frames, wa)
    lc = batch_center(landmarks, wa)
    out = np.empty((frames.shape[0], landmarks.shape[0]))
    for t0 in range(0, frames.shape[0], block):
        vals, _, _, _ = batch_fit(fc[t0:t0 + block, None], lc[None], w)
        out[t0:t0 + block] = vals[..., 0]
    return out


def _batch_cv(dist, q, lam, dgrads_fn):
    """s, z and their gradients from D [L] and a callable giving sum_i c_i dD_i."""
    dmin = dist.min()
    e = np.exp(-lam * (dist - dmin))
    zsum = e.sum()
    p = e / zsum
    s = float(p @ q)
    z = float(dmin - math.log(zsum) / lam)
    if dgrads_fn is None:
        return s, z, None, None
    cs = -lam * p * (q - s)
    return s, z, dgrads_fn(cs), dgrads_fn(p)


def batch_path_cv_exact(frames, landmarks, lam, q=None, w=None, w_align=None, grad=True):
    """Vectorised Alg. 1: exact D, s, z, ds, dz (dR term dropped: it is zero
    at the optimum; the per-pair oracle keeps it and the CPU
    tests show the two agree)."""
    frames = np.asarray(frames, dtype=float)
    landmarks = np.asarray(landmarks, dtype=float)
    t_count, n, _ = frames.shape
    n_l = landmarks.shape[0]
    w = normalise_weights(w, n)
    wa = normalise_weights(w_align, n)
    q = np.arange(n_l, dtype=float) if q is None else np.asarray(q, dtype=float)
    fc = batch_center(frames, wa)
    lc = batch_center(landmarks, wa)
    out = {"s": np.zeros(t_count), "z": np.zeros(t_count), "D": np.zeros((t_count, n_l))}
    if grad:
        out["ds"] = np.zeros((t_count, n, 3))
        out["dz"] = np.zeros((t_count, n, 3))
    for t in range(t_count):
        vals, _, rot, _ = batch_fit(fc[t][None], lc, w)
        dist = vals[:, 0]
        out["D"][t] = dist
        ra = np.einsum("iab,ijb->ija", rot, lc)  # R_i a_i

        def dg(c, xc=fc[t], ra=ra):
            g = 2.0 * w[:, None] * (c.sum() * xc - np.einsum("i,ija->ja", c, ra))
            return _uncenter(g, wa)

        s, z, ds, dz = _batch_cv(dist, q, lam, dg if grad else None)
        out["s"][t], out["z"][t] = s, z
        if grad:
            out["ds"][t], out["dz"][t] = ds, dz
    return out


# --------------------------------------------------------------------------
# Metadynamics bias and force (SPEC [MODULE] metadynamics; PAPER Eq. 1;
# SURVEY §8(f) 2).  Test infrastructure only, like everything in oracle/.
# --------------------------------------------------------------------------

def mtd_bias_direct(cv, centers, sigmas, heights):
    """V(S) = sum_h w_h prod_i exp(-(S_i - c_hi)^2 / (2 sigma_hi^2)) and dV/dS_i
    (analytic hill derivative; SPEC metadynamics bias_and_force, direct mode).
    cv [T, d]; centers, sigmas [H, d]; heights [H] -> V [T], dV [T, d]."""
    cv = np.atleast_2d(np.asarray(cv, dtype=float))
    centers = np.asarray(centers, dtype=float).reshape(-1, cv.shape[1])
    sigmas = np.asarray(sigmas, dtype=float).reshape(-1, cv.shape[1])
    heights = np.asarray(heights, dtype=float).reshape(-1)
    if centers.shape[0] == 0:
        return np.zeros(cv.shape[0]), np.zeros_like(cv)
    u = (cv[:, None, :] - centers[None]) / sigmas[None]          # [T, H, d]
    g = heights[None] * np.exp(-0.5 * np.sum(u * u, axis=-1))     # [T, H]
    V = g.sum(axis=1)
    dV = np.einsum("th,thd->td", g, -u / sigmas[None])
    return V, dV


def mtd_grid_new(lo, hi, bins):
    """Uniform grid per CV dimension (SPEC HillStore.grid): nodes lo + k h, k = 0..bins.
    Stores values, first derivatives per dimension and (d = 2) the cross derivative,
    the data of a tensor-product cubic Hermite interpolant."""
    lo, hi = np.atleast_1d(np.asarray(lo, float)), np.atleast_1d(np.asarray(hi, float))
    bins = np.atleast_1d(np.asarray(bins, int))
    d = lo.shape[0]
    if d not in (1, 2) or hi.shape != lo.shape or bins.shape != lo.shape or np.any(hi <= lo) or np.any(bins < 1):
        raise ValueError("grid: 1 or 2 dimensions with lo < hi and bins >= 1")
    shape = tuple(int(b) + 1 for b in bins)
    return {"lo": lo, "hi": hi, "bins": bins, "h": (hi - lo) / bins, "val": np.zeros(shape),
            "d": [np.zeros(shape) for _ in range(d)], "dxy": np.zeros(shape) if d == 2 else None}


def mtd_grid_deposit(grid, center, sigma, height, cutoff=6.0):
    """Add one hill to every grid node within `cutoff` sigmas per dimension (SPEC:
    truncation radius 6 sigma, error <= w e^-18).  Out-of-grid centre -> error."""
    c, s = np.atleast_1d(np.asarray(center, float)), np.atleast_1d(np.asarray(sigma, float))
    if np.any(c < grid["lo"]) or np.any(c > grid["hi"]):
        raise ValueError("hill centre outside the grid")
    axes = [grid["lo"][i] + grid["h"][i] * np.arange(grid["bins"][i] + 1) for i in range(c.shape[0])]
    masks = [np.abs(ax - c[i]) <= cutoff * s[i] for i, ax in enumerate(axes)]
    u = [np.where(m, (ax - c[i]) / s[i], 0.0) for i, (ax, m) in enumerate(zip(axes, masks))]
    e = [np.where(m, np.exp(-0.5 * ui * ui), 0.0) for ui, m in zip(u, masks)]
    if c.shape[0] == 1:
        g = height * e[0]
        grid["val"] += g
        grid["d"][0] += g * (-u[0] / s[0])
    else:
        g = height * np.outer(e[0], e[1])
        a0, a1 = (-u[0] / s[0])[:, None], (-u[1] / s[1])[None, :]
        grid["val"] += g
        grid["d"][0] += g * a0
        grid["d"][1] += g * a1
        grid["dxy"] += g * a0 * a1
    return grid


def _hermite(t):
    t2, t3 = t * t, t * t * t
    return (2 * t3 - 3 * t2 + 1, -2 * t3 + 3 * t2, t3 - 2 * t2 + t, t3 - t2,
            6 * t2 - 6 * t, -6 * t2 + 6 * t, 3 * t2 - 4 * t + 1, 3 * t2 - 2 * t)


def mtd_grid_eval(grid, cv):
    """Cubic Hermite interpolation (per dimension; tensor product for d = 2) of the
    grid values -> V [T], dV [T, d].  A CV outside the grid raises ValueError (SPEC:
    out-of-grid error)."""
    cv = np.atleast_2d(np.asarray(cv, dtype=float))
    d = cv.shape[1]
    if np.any(cv < grid["lo"]) or np.any(cv > grid["hi"]):
        raise ValueError("collective variable outside the bias grid")
    idx, tt = [], []
    for i in range(d):
        x = (cv[:, i] - grid["lo"][i]) / grid["h"][i]
        k = np.minimum(np.floor(x).astype(int), grid["bins"][i] - 1)
        idx.append(k)
        tt.append(x - k)
    V = np.zeros(cv.shape[0])
    dV = np.zeros_like(cv)
    if d == 1:
        k, t, h = idx[0], tt[0], grid["h"][0]
        h00, h01, h10, h11, d00, d01, d10, d11 = _hermite(t)
        f0, f1 = grid["val"][k], grid["val"][k + 1]
        g0, g1 = grid["d"][0][k] * h, grid["d"][0][k + 1] * h
        V = h00 * f0 + h01 * f1 + h10 * g0 + h11 * g1
        dV[:, 0] = (d00 * f0 + d01 * f1 + d10 * g0 + d11 * g1) / h
        return V, dV
    kx, ky, tx, ty = idx[0], idx[1], tt[0], tt[1]
    hx, hy = grid["h"]
    bx, by = _hermite(tx), _hermite(ty)
    for a in (0, 1):
        for b in (0, 1):
            f = grid["val"][kx + a, ky + b]
            fx = grid["d"][0][kx + a, ky + b] * hx
            fy = grid["d"][1][kx + a, ky + b] * hy
            fxy = grid["dxy"][kx + a, ky + b] * hx * hy
            H0x, H1x, D0x, D1x = bx[a], bx[2 + a], bx[4 + a], bx[6 + a]
            H0y, H1y, D0y, D1y = by[b], by[2 + b], by[4 + b], by[6 + b]
            V += f * H0x * H0y + fx * H1x * H0y + fy * H0x * H1y + fxy * H1x * H1y
            dV[:, 0] += (f * D0x * H0y + fx * D1x * H0y + fy * D0x * H1y + fxy * D1x * H1y) / hx
            dV[:, 1] += (f * H0x * D0y + fx * H1x * D0y + fy * H0x * D1y + fxy * H1x * D1y) / hy
    return V, dV


def mtd_force(dV, grads):
    """Bias force on the atoms (SPEC: F = -dV/dx, the physical sign; Eq. 1 prints +):
    F_k = -sum_i (dV/dS_i) (dS_i/dx_k).  dV [T, d]; grads: d arrays [T, N, 3]."""
    dV = np.asarray(dV, dtype=float)
    return -sum(dV[:, i, None, None] * np.asarray(g, dtype=float) for i, g in enumerate(grads))
