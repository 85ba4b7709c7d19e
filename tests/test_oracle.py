"""Pin the CPU oracle to the reference (golden vectors) and to the SPEC KATs.

These run without a GPU.  The golden vectors come from the reference
implementation itself (tests/golden/make_golden.py).
"""

import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1801_02362_b200 import synth


def _fits(golden):
    g = golden("fits.npz")
    for i in range(int(g["count"])):
        yield {k.split("_", 1)[1]: g[k] for k in g.files if k.startswith(f"{i}_")}


def test_center_matches_reference(golden):
    for c in _fits(golden):
        wa = O.normalise_weights(c["wa"], int(c["n"]))
        np.testing.assert_allclose(O.center(c["x"], wa), c["xc"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(O.center(c["a"], wa), c["ac"], rtol=0, atol=1e-15)


def test_kearsley_fit_matches_reference(golden):
    n_checked = 0
    for c in _fits(golden):
        fit = O.kearsley_fit(c["xc"], c["ac"], c["w"], with_derivatives=False)
        np.testing.assert_allclose(fit["eigvals"], c["eigvals"], rtol=0, atol=1e-13)
        if c["kind"] in ("same", "rotated"):
            # x == a and x == Q a: eigvals[0] is zero; quaternion may sit on a
            # degenerate pair only in the symmetric cases - compare R only
            np.testing.assert_allclose(fit["rot"], c["rot"], atol=1e-9)
        else:
            np.testing.assert_allclose(fit["quat"], c["quat"], atol=1e-12)
            np.testing.assert_allclose(fit["rot"], c["rot"], atol=1e-12)
        if not bool(c["degenerate"]):
            fd = O.kearsley_fit(c["xc"], c["ac"], c["w"], with_derivatives=True)
            scale = max(1.0, float(np.abs(c["rot_grad"]).max()))
            np.testing.assert_allclose(fd["rot_grad"] / scale, c["rot_grad"] / scale, atol=1e-10)
        n_checked += 1
    assert n_checked == 80


def test_jacobi_matches_reference(golden):
    g = golden("jacobi.npz")
    for m, v, vec in zip(g["mats"], g["vals"], g["vecs"]):
        w, u = O.jacobi_eigh(m)
        scale = max(1.0, np.abs(m).max())
        np.testing.assert_allclose(w / scale, v / scale, atol=1e-13)
        np.testing.assert_allclose(u, vec, atol=1e-9)


def _jacobi_n_cases(g):
    """Unpack tests/golden/jacobi_n.npz (flat per-field arrays) into per-case tuples."""
    o1 = o2 = 0
    for n, tol, ms, ok in zip(g["sizes"], g["tols"], g["sweeps"], g["conv"]):
        n = int(n)
        m = g["mats"][o2:o2 + n * n].reshape(n, n)
        v = g["vals"][o1:o1 + n]
        u = g["vecs"][o2:o2 + n * n].reshape(n, n)
        o1 += n
        o2 += n * n
        yield m, float(tol), int(ms), bool(ok), v, u


def test_jacobi_general_n_matches_reference(golden):
    """The oracle's jacobi_eigh on the reference's general-size cases (n = 1..40, custom
    tolerances, sweep limits that make the reference raise RuntimeError)."""
    for m, tol, ms, ok, v, u in _jacobi_n_cases(golden("jacobi_n.npz")):
        if not ok:
            with pytest.raises(RuntimeError):
                O.jacobi_eigh(m, tol=tol, max_sweeps=ms)
            continue
        w, vec = O.jacobi_eigh(m, tol=tol, max_sweeps=ms)
        scale = max(1.0, np.abs(m).max())
        np.testing.assert_allclose(w / scale, v / scale, atol=1e-12)
        np.testing.assert_allclose(vec, u, atol=1e-8)


def test_misc_reference_cases(golden):
    g = golden("misc.npz")
    w = np.full(8, 1 / 8)
    val = O.rotation_derivative_check(g["check_x"], g["check_a"], w)
    assert val < 1e-5
    assert abs(val - float(g["check_value"])) < 1e-7
    w2 = np.full(2, 0.5)
    fit = O.kearsley_fit(g["deg_x"], g["deg_a"], w2)
    np.testing.assert_allclose(fit["eigvals"], g["deg_eigvals"], atol=1e-14)
    assert bool(g["deg_raised"])
    with pytest.raises(O.DegenerateFit):
        O.kearsley_fit(g["deg_x"], g["deg_a"], w2, with_derivatives=True)


def test_pathcv0_distances_and_rotations(golden):
    g = golden("pathcv0.npz")
    n = g["frames"].shape[1]
    w = np.full(n, 1.0 / n)
    for t in range(g["frames"].shape[0]):
        xc = O.center(g["frames"][t], w)
        np.testing.assert_allclose(xc, g["xc"][t], atol=1e-15)
        for i in range(g["landmarks"].shape[0]):
            d, grad, fit = O.exact_distance(xc, g["lc"][i], w, w)
            assert abs(d - g["D"][t, i]) <= 1e-13 * max(1.0, g["D"][t, i])
            np.testing.assert_allclose(fit["rot"], g["R"][t, i], atol=1e-12)


def test_pathcv0_full_chain_against_reference_fits(golden):
    """s, z and gradients assembled from the reference's own fits (Eq. 4 literal)."""
    g = golden("pathcv0.npz")
    frames, lms, lam = g["frames"], g["landmarks"], float(g["lam"])
    n = frames.shape[1]
    L = lms.shape[0]
    w = np.full(n, 1.0 / n)
    q = np.arange(L, dtype=float)
    out = O.path_cv_exact(frames, lms, lam)
    for t in range(frames.shape[0]):
        # reference-built gradient of every D_i (2 w d + dR term, then w' term)
        grads = np.zeros((L, n, 3))
        for i in range(L):
            d = g["xc"][t] - g["lc"][i] @ g["R"][t, i].T
            mm = -2.0 * (w[:, None] * d).T @ g["lc"][i]
            gg = 2.0 * w[:, None] * d + np.einsum("bg,kabg->ka", mm, g["rot_grad"][t, i])
            grads[i] = gg - w[:, None] * gg.sum(axis=0)
        dist = g["D"][t]
        e = np.exp(-lam * (dist - dist.min()))
        p = e / e.sum()
        s = p @ q
        z = dist.min() - math.log(e.sum()) / lam
        ds = np.einsum("i,ika->ka", -lam * p * (q - s), grads)
        dz = np.einsum("i,ika->ka", p, grads)
        assert abs(out["s"][t] - s) <= 1e-10 * max(1, abs(s))
        assert abs(out["z"][t] - z) <= 1e-12
        np.testing.assert_allclose(out["ds"][t], ds, atol=1e-8 * np.abs(ds).max())
        np.testing.assert_allclose(out["dz"][t], dz, atol=1e-8 * np.abs(dz).max())


def test_close_structure_against_reference_run(golden):
    g = golden("close.npz")
    out = O.close_structure_replay(g["frames"], g["landmarks"], lam=100.0, eps=float(g["eps"]),
                                   grad=False)
    np.testing.assert_array_equal(out["refresh"], g["refresh"])
    np.testing.assert_allclose(out["dxy"], g["dxy"], rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(out["D"], g["D"], rtol=1e-10, atol=1e-15)
    assert 0 < g["refresh"].sum() < len(g["refresh"])
    c = out["counters"]
    T, L = g["frames"].shape[0], g["landmarks"].shape[0]
    assert c["expensive_count"] == T + c["reassign_count"] * L
    assert c["cheap_count"] == (T - c["reassign_count"]) * L


# ---------------------------------------------------------------- SPEC KATs

def test_spec_fit_identity_and_rotation():
    rng = np.random.default_rng(5)
    a = O.center(rng.normal(size=(6, 3)), np.full(6, 1 / 6))
    w = np.full(6, 1 / 6)
    fit = O.kearsley_fit(a, a, w)
    np.testing.assert_allclose(fit["rot"], np.eye(3), atol=1e-12)
    assert abs(fit["eigvals"][0]) < 1e-14
    qrot = synth.random_rotations(rng, 1)[0]
    fit = O.kearsley_fit(a @ qrot.T, a, w)
    np.testing.assert_allclose(fit["rot"], qrot, atol=1e-10)
    assert abs(fit["eigvals"][0]) < 1e-10
    r = fit["rot"]
    np.testing.assert_allclose(r.T @ r, np.eye(3), atol=1e-10)
    assert abs(np.linalg.det(r) - 1) < 1e-10


def test_spec_eigval_equals_eq3_sum():
    rng = np.random.default_rng(6)
    for n in (3, 7, 12):
        w = O.normalise_weights(rng.uniform(0.1, 1, n), n)
        wa = O.normalise_weights(rng.uniform(0.1, 1, n), n)
        x = O.center(rng.normal(size=(n, 3)), wa)
        a = O.center(rng.normal(size=(n, 3)), wa)
        fit = O.kearsley_fit(x, a, w)
        d = x - a @ fit["rot"].T
        assert abs(np.sum(w * np.sum(d * d, 1)) - fit["eigvals"][0]) <= 1e-10 * fit["eigvals"][0]


def test_spec_exact_gradient_fd():
    """Eq. 4 gradient vs central differences of D, w != w'."""
    rng = np.random.default_rng(7)
    n = 6
    w = O.normalise_weights(rng.uniform(0.1, 1, n), n)
    wa = O.normalise_weights(rng.uniform(0.1, 1, n), n)
    x = rng.normal(scale=0.3, size=(n, 3))
    a = O.center(rng.normal(scale=0.3, size=(n, 3)), wa)

    def dist(xr):
        return O.kearsley_fit(O.center(xr, wa), a, w)["eigvals"][0]

    _, g, _ = O.exact_distance(O.center(x, wa), a, w, wa)
    h = 1e-6
    fd = np.zeros_like(x)
    for k in range(n):
        for al in range(3):
            xp, xm = x.copy(), x.copy()
            xp[k, al] += h
            xm[k, al] -= h
            fd[k, al] = (dist(xp) - dist(xm)) / (2 * h)
    assert np.abs(fd - g).max() <= 1e-5 * np.abs(g).max()
    assert np.abs(g.sum(axis=0)).max() < 1e-8


def test_spec_approx_gradient_fd_and_identity():
    """Eq. 5/6: FD and approx == exact at y = x."""
    rng = np.random.default_rng(8)
    n = 6
    w = O.normalise_weights(rng.uniform(0.1, 1, n), n)
    wa = O.normalise_weights(rng.uniform(0.1, 1, n), n)
    y = O.center(rng.normal(scale=0.3, size=(n, 3)), wa)
    a = O.center(rng.normal(scale=0.3, size=(n, 3)), wa)
    rot_ay = O.kearsley_fit(y, a, w)["rot"]
    fit_yy = O.kearsley_fit(y, y, w, with_derivatives=True)
    v_approx, _ = O.approx_distance(y, a, rot_ay, fit_yy, w, wa)
    v_exact, _, _ = O.exact_distance(y, a, w, wa)
    assert abs(v_approx - v_exact) < 1e-12
    x = y + rng.normal(scale=0.01, size=(n, 3))

    def dist(xr):
        xc = O.center(xr, wa)
        return O.approx_distance(xc, a, rot_ay, O.kearsley_fit(xc, y, w, with_derivatives=True), w, wa)[0]

    xc = O.center(x, wa)
    _, g = O.approx_distance(xc, a, rot_ay, O.kearsley_fit(xc, y, w, with_derivatives=True), w, wa)
    h = 1e-6
    fd = np.zeros_like(x)
    for k in range(n):
        for al in range(3):
            xp, xm = x.copy(), x.copy()
            xp[k, al] += h
            xm[k, al] -= h
            fd[k, al] = (dist(xp) - dist(xm)) / (2 * h)
    assert np.abs(fd - g).max() <= 1e-5 * np.abs(g).max()
    assert np.abs(g.sum(axis=0)).max() < 1e-8


def test_spec_property_map_kats():
    s, ds = O.property_map([0.3], np.zeros((1, 2, 3)) + 1.0, [4.0], 7.0)
    assert s == 4.0 and np.all(ds == 0)
    s, _ = O.property_map([0.2, 0.2], None, [1.0, 2.0], 3.0)
    assert abs(s - 1.5) < 1e-15
    import mpmath  # high-precision Eq. 2

    mpmath.mp.dps = 50
    d = [mpmath.mpf("0.01"), mpmath.mpf("0.5")]
    qv = [3, 7]
    num = sum(qq * mpmath.e ** (-10 * dd) for qq, dd in zip(qv, d))
    den = sum(mpmath.e ** (-10 * dd) for dd in d)
    s, _ = O.property_map([0.01, 0.5], None, qv, 10.0)
    assert abs(s - float(num / den)) < 1e-12
    s1, _ = O.property_map([0.01, 0.5, 0.2], None, [1, 2, 3], 10.0)
    s2, _ = O.property_map([1.01, 1.5, 1.2], None, [1, 2, 3], 10.0)
    assert abs(s1 - s2) < 1e-12
    s, _ = O.property_map([0.1, 0.2, 0.3], None, [5, 6, 7], 1000.0)
    assert abs(s - 5.0) < 1e-10


def test_spec_pathcv_chain_fd():
    """Full-chain gradient of s and z vs FD: 6 atoms, 4 refs."""
    rng = np.random.default_rng(9)
    n, L = 6, 4
    lms = rng.normal(scale=0.3, size=(L, n, 3))
    x = lms[1] + rng.normal(scale=0.05, size=(n, 3))
    lam = 5.0
    out = O.path_cv_exact(x[None], lms, lam)
    h = 1e-6
    fds, fdz = np.zeros_like(x), np.zeros_like(x)
    for k in range(n):
        for al in range(3):
            xp, xm = x.copy(), x.copy()
            xp[k, al] += h
            xm[k, al] -= h
            op = O.path_cv_exact(xp[None], lms, lam, grad=False)
            om = O.path_cv_exact(xm[None], lms, lam, grad=False)
            fds[k, al] = (op["s"][0] - om["s"][0]) / (2 * h)
            fdz[k, al] = (op["z"][0] - om["z"][0]) / (2 * h)
    assert np.abs(fds - out["ds"][0]).max() <= 1e-5 * np.abs(out["ds"][0]).max()
    assert np.abs(fdz - out["dz"][0]).max() <= 1e-5 * np.abs(out["dz"][0]).max()


def test_eps_zero_equals_exact():
    """eps -> 0 reassigns every frame, results are exact."""
    wl = synth.config0(seed=3, T=6, L=5, N=7)
    ex = O.path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    cl = O.close_structure_replay(wl.frames, wl.landmarks, wl.lam, eps=0.0)
    assert cl["refresh"].all()
    np.testing.assert_allclose(cl["s"], ex["s"], rtol=1e-12)
    np.testing.assert_allclose(cl["ds"], ex["ds"], atol=1e-12)


def test_batch_oracle_matches_per_pair():
    wl = synth.config0(seed=4, T=5, L=7, N=9)
    per = O.path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    bat = O.batch_path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    np.testing.assert_allclose(bat["D"], per["D"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(bat["s"], per["s"], rtol=1e-12)
    np.testing.assert_allclose(bat["z"], per["z"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(bat["ds"], per["ds"], atol=1e-10 * np.abs(per["ds"]).max())
    np.testing.assert_allclose(bat["dz"], per["dz"], atol=1e-10 * np.abs(per["dz"]).max())
    m = O.batch_msd_matrix(wl.frames, wl.landmarks)
    np.testing.assert_allclose(m, per["D"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("seed,eps_mult", [(3, 1.0), (5, 4.0)])
def test_close_lifetime_window_contains_every_needed_landmark(seed, eps_mult):
    """The certificate behind the pruned close-structure replay (engine.PathCV
    ._close_replay_pruned, csrc/refine.cu cand_kernel): for a refresh frame y with lifetime
    bound delta = max D(x, y) over the frames x that keep y, every landmark any such x needs
    (lam (D~_l(x) - min D~(x)) <= thr, Eq. 5 distances) satisfies
    d(y, a_l) <= sqrt(delta) + sqrt((sqrt(delta) + d_min(y))^2 + thr / lam)  (RMSD triangle
    inequality).  Checked with the oracle's exact and Eq. 5 distances on a config-3-like
    walker (accumulated noise), every frame, every landmark."""
    wl = synth.config3(seed=seed, W=1, N=40, L=60, steps=120)
    frames = wl.frames[0].astype(np.float64)
    lm = wl.landmarks.astype(np.float64)
    eps = wl.eps * eps_mult
    out = O.close_structure_replay(frames, lm, wl.lam, eps, grad=False)
    ref, D, dxy = out["refresh"], out["D"], out["dxy"]
    assert ref[0] and 0 < ref.sum() < len(ref)
    ridx = np.maximum.accumulate(np.where(ref, np.arange(len(ref)), 0))
    thr = 27.0
    checked = 0
    for y in np.nonzero(ref)[0]:
        life = np.nonzero((ridx == y) & ~ref)[0]
        delta = dxy[life].max() if life.size else 0.0
        dy = np.sqrt(np.maximum(D[y], 0.0))  # refresh row: exact distances of y
        bound = np.sqrt(delta) + np.sqrt((np.sqrt(delta) + dy.min()) ** 2 + thr / wl.lam)
        inside = dy <= bound * (1 + 1e-12)
        for x in np.concatenate([[y], life]):
            need = wl.lam * (D[x] - D[x].min()) <= thr
            assert np.all(inside[need]), (y, x)
            checked += int(need.sum())
    assert checked > 0
