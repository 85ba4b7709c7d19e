"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``metadyn_close.geometry`` from /root/reference/pkg/src and writes
small ``.npz`` fixtures next to this script.  The fixtures are committed; the
GPU box never reads /root/reference.

Contents
* ``fits.npz``      kearsley_fit (rot, quat, eigvals, rot_grad) + Structure
                    centring for seeded pairs: N in {2..12, 22, 304}, random
                    and uniform weights, x == a, x = Q a, near-identical pairs.
* ``jacobi.npz``    jacobi_eigh on random symmetric 4x4 matrices.
* ``jacobi_n.npz``  jacobi_eigh on symmetric n x n matrices (n = 1..40, several
                    tolerances / sweep limits); entries with ``conv`` = 0 raised
                    RuntimeError (not enough sweeps).
* ``misc.npz``      rotation_derivative_check on an 8-atom pair, the degenerate
                    2-atom case (DegenerateFitError) and error cases.
* ``pathcv0.npz``   a config-0-shaped slice (8 frames x 20 landmarks x 22
                    atoms): per-pair reference fits (eigvals[0], rot, rot_grad)
                    for every (frame, landmark) pair, centred via Structure.
* ``close.npz``     a small close-structure run (30 frames x 6 landmarks x 12
                    atoms) whose fits (x<->y with derivatives, y<->a_i) all come
                    from the reference ``kearsley_fit``.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from metadyn_close import errors as ref_errors  # noqa: E402
from metadyn_close import geometry as ref  # noqa: E402

from paper_1801_02362_b200 import synth  # noqa: E402


def _fit_case(rng, n, weighted, kind):
    a = rng.normal(0.0, 0.3, size=(n, 3))
    if kind == "random":
        x = rng.normal(0.0, 0.3, size=(n, 3))
    elif kind == "noisy":
        x = a + rng.normal(0.0, 0.05, size=(n, 3))
    elif kind == "near":
        x = a + rng.normal(0.0, 1e-4, size=(n, 3))
    elif kind == "same":
        x = a.copy()
    else:  # rotated copy
        x = a.copy()
    rot = synth.random_rotations(rng, 1)[0]
    trans = rng.uniform(-1, 1, size=3)
    x = x @ rot.T + trans
    a = a + rng.uniform(-1, 1, size=3)
    w = rng.uniform(0.1, 1.0, size=n) if weighted else None
    wa = rng.uniform(0.1, 1.0, size=n) if weighted else None
    return x, a, w, wa


def make_fits(rng):
    rows = []
    specs = []
    for n in (3, 4, 5, 6, 8, 12, 22, 304):
        for weighted in (False, True):
            for kind in ("random", "noisy", "near", "same", "rotated"):
                specs.append((n, weighted, kind))
    for n, weighted, kind in specs:
        x, a, w, wa = _fit_case(rng, n, weighted, kind)
        sx = ref.Structure(x, w, wa)
        sa = ref.Structure(a, w, wa)
        xc, ac = sx.center(), sa.center()
        try:
            fit = ref.kearsley_fit(xc, ac, with_derivatives=True)
            rot_grad = fit.rot_grad
            degenerate = False
        except ref_errors.DegenerateFitError:
            fit = ref.kearsley_fit(xc, ac)
            rot_grad = np.zeros((n, 3, 3, 3))
            degenerate = True
        rows.append(dict(
            n=n, x=x, a=a, w=sx.disp_weights, wa=sx.align_weights,
            xc=xc.coords, ac=ac.coords, rot=fit.rot, quat=fit.quat,
            eigvals=fit.eigvals, rot_grad=rot_grad, degenerate=degenerate,
            kind=kind, weighted=weighted,
        ))
    out = {"count": len(rows)}
    for i, r in enumerate(rows):
        for k, v in r.items():
            out[f"{i}_{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "fits.npz"), **out)
    return len(rows)


def make_jacobi(rng):
    mats, vals, vecs = [], [], []
    for i in range(64):
        b = rng.normal(size=(4, 4)) * (10.0 ** rng.uniform(-3, 3))
        m = b + b.T
        if i % 8 == 0:
            m = np.diag(rng.normal(size=4))  # already diagonal
        w, v = ref.jacobi_eigh(m)
        mats.append(m)
        vals.append(w)
        vecs.append(v)
    np.savez_compressed(os.path.join(HERE, "jacobi.npz"), mats=np.array(mats),
                        vals=np.array(vals), vecs=np.array(vecs))


def make_jacobi_n(rng):
    """General-size cases for the device jacobi_eigh: one flat array per field."""
    sizes, tols, sweeps, mats, vals, vecs, conv = [], [], [], [], [], [], []
    cases = [(n, 1e-14, 60) for n in (1, 2, 3, 5, 6, 7, 9, 12, 16, 20, 33, 40)]
    cases += [(4, 1e-8, 60), (6, 1e-6, 60), (8, 1e-14, 2), (10, 1e-14, 1), (5, 0.0, 60)]
    for n, tol, ms in cases:
        b = rng.normal(size=(n, n)) * (10.0 ** rng.uniform(-2, 2))
        m = b + b.T
        try:
            w, v = ref.jacobi_eigh(m, tol=tol, max_sweeps=ms)
            ok = 1
        except RuntimeError:
            w, v, ok = np.zeros(n), np.zeros((n, n)), 0
        sizes.append(n)
        tols.append(tol)
        sweeps.append(ms)
        mats.append(m.ravel())
        vals.append(w.ravel())
        vecs.append(v.ravel())
        conv.append(ok)
    np.savez_compressed(os.path.join(HERE, "jacobi_n.npz"), sizes=np.array(sizes), tols=np.array(tols),
                        sweeps=np.array(sweeps), conv=np.array(conv), mats=np.concatenate(mats),
                        vals=np.concatenate(vals), vecs=np.concatenate(vecs))


def make_misc(rng):
    x, a, _, _ = _fit_case(rng, 8, False, "random")
    sx, sa = ref.Structure(x).center(), ref.Structure(a).center()
    check = ref.rotation_derivative_check(sx, sa, h=1e-6)
    # two atoms: rotation about the bond axis is free -> degenerate spectrum
    x2 = np.array([[0.0, 0.0, 0.5], [0.0, 0.0, -0.5]])
    a2 = np.array([[0.3, 0.0, 0.0], [-0.3, 0.0, 0.0]])
    s2x, s2a = ref.Structure(x2).center(), ref.Structure(a2).center()
    fit2 = ref.kearsley_fit(s2x, s2a)
    try:
        ref.kearsley_fit(s2x, s2a, with_derivatives=True)
        degenerate_raised = False
    except ref_errors.DegenerateFitError:
        degenerate_raised = True
    np.savez_compressed(
        os.path.join(HERE, "misc.npz"), check_x=sx.coords, check_a=sa.coords,
        check_value=check, deg_x=s2x.coords, deg_a=s2a.coords, deg_eigvals=fit2.eigvals,
        deg_raised=degenerate_raised)


def make_pathcv0():
    wl = synth.config0(seed=0)
    frames = wl.frames[:8]
    lms = wl.landmarks
    T, L, N = frames.shape[0], lms.shape[0], frames.shape[1]
    D = np.zeros((T, L))
    R = np.zeros((T, L, 3, 3))
    RG = np.zeros((T, L, N, 3, 3, 3))
    lc = [ref.Structure(a).center() for a in lms]
    xcs = []
    for t in range(T):
        xc = ref.Structure(frames[t]).center()
        xcs.append(xc.coords)
        for i in range(L):
            fit = ref.kearsley_fit(xc, lc[i], with_derivatives=True)
            D[t, i] = fit.eigvals[0]
            R[t, i] = fit.rot
            RG[t, i] = fit.rot_grad
    np.savez_compressed(os.path.join(HERE, "pathcv0.npz"), frames=frames, landmarks=lms,
                        xc=np.array(xcs), lc=np.array([s.coords for s in lc]), lam=wl.lam,
                        D=D, R=R, rot_grad=RG)


def make_close():
    """Small Alg. 2 run with every fit done by the reference kearsley_fit."""
    rng = np.random.default_rng(11)
    N, L, T = 12, 6, 30
    ends = rng.normal(0.0, 0.3, size=(2, N, 3))
    lms = synth.make_landmarks(rng, ends, L, noise=0.01)
    # slow drift along the path with small accumulated noise so that both
    # refresh and approximate frames occur
    p = np.linspace(0.5, 1.5, T)
    base = synth.path_points(ends, p, L)
    noise = np.cumsum(rng.normal(0.0, 0.002, size=(T, N, 3)), axis=0)
    frames = synth.rigid_motion(rng, base + noise)
    eps = 2e-4
    lc = [ref.Structure(a).center() for a in lms]
    y = None
    saved = [None] * L
    refresh = np.zeros(T, dtype=bool)
    dxy = np.zeros(T)
    D = np.zeros((T, L))
    rxy = np.zeros((T, 3, 3))
    rxy_grad = np.zeros((T, N, 3, 3, 3))
    saved_log = np.zeros((T, L, 3, 3))
    for t in range(T):
        xc = ref.Structure(frames[t]).center()
        if y is None:
            fresh = True
        else:
            fit_xy = ref.kearsley_fit(xc, y, with_derivatives=True)
            dxy[t] = fit_xy.eigvals[0]
            rxy[t] = fit_xy.rot
            rxy_grad[t] = fit_xy.rot_grad
            fresh = fit_xy.eigvals[0] > eps
        refresh[t] = fresh
        if fresh:
            y = xc
            for i in range(L):
                fit = ref.kearsley_fit(xc, lc[i])
                saved[i] = fit.rot
                D[t, i] = fit.eigvals[0]
        else:
            w = xc.disp_weights
            for i in range(L):
                b = lc[i].coords @ saved[i].T
                d = xc.coords - b @ fit_xy.rot.T
                D[t, i] = np.sum(w * np.sum(d * d, axis=1))
        saved_log[t] = np.array(saved)
    np.savez_compressed(os.path.join(HERE, "close.npz"), frames=frames, landmarks=lms, eps=eps,
                        refresh=refresh, dxy=dxy, D=D, rxy=rxy, rxy_grad=rxy_grad,
                        saved=saved_log)
    return int(refresh.sum())


def main():
    rng = np.random.default_rng(20180107)
    n = make_fits(rng)
    make_jacobi(rng)
    make_jacobi_n(np.random.default_rng(1234))
    make_misc(rng)
    make_pathcv0()
    k = make_close()
    print(f"fits: {n} cases; close run refreshes: {k}/30")


if __name__ == "__main__":
    main()
