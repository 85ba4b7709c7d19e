"""GPU tests of the reference-facing API (geometry / msd / colvar mirrors),
read like the reference's own SPEC examples, against the reference golden
vectors and the CPU oracle."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_1801_02362_b200 import colvar, errors, geometry as G, msd, synth

pytestmark = pytest.mark.gpu


def _fits(golden):
    g = golden("fits.npz")
    for i in range(int(g["count"])):
        yield {k.split("_", 1)[1]: g[k] for k in g.files if k.startswith(f"{i}_")}


def test_structure_validation_matches_reference():
    with pytest.raises(errors.InvalidStructureError):
        G.Structure(np.zeros((1, 3)))
    with pytest.raises(errors.InvalidStructureError):
        G.Structure(np.zeros((3, 2)))
    with pytest.raises(errors.InvalidStructureError):
        G.Structure([[0, 0, np.nan], [1, 1, 1]])
    with pytest.raises(errors.InvalidStructureError):
        G.Structure(np.zeros((2, 3)), disp_weights=[0.0, 0.0])
    s = G.Structure(np.eye(3), disp_weights=[1, 1, 2])
    np.testing.assert_allclose(s.disp_weights, [0.25, 0.25, 0.5])
    assert not s.coords.flags.writeable


def test_center_matches_reference_golden(golden, cuda_device):
    for c in list(_fits(golden))[::3]:
        s = G.Structure(c["x"], c["w"], c["wa"])
        np.testing.assert_allclose(s.center().coords, c["xc"], atol=1e-14)
        assert s.center().is_centered()
    # SPEC.md:49-51 examples
    np.testing.assert_allclose(G.center(G.Structure([[2, 0, 0], [0, 0, 0]])).coords, [[1, 0, 0], [-1, 0, 0]])
    np.testing.assert_allclose(G.Structure([[1, 0, 0], [-1, 0, 0]]).center().coords, [[1, 0, 0], [-1, 0, 0]])


def test_kearsley_fit_matches_reference_golden(golden, cuda_device):
    for c in _fits(golden):
        x = G.Structure(c["xc"], c["w"], c["wa"])
        a = G.Structure(c["ac"], c["w"], c["wa"])
        deg = bool(c["degenerate"])
        if deg:
            with pytest.raises(errors.DegenerateFitError):
                G.kearsley_fit(x, a, with_derivatives=True)
            fit = G.kearsley_fit(x, a)
        else:
            fit = G.kearsley_fit(x, a, with_derivatives=True)
            scale = max(1.0, np.abs(c["rot_grad"]).max())
            np.testing.assert_allclose(fit.rot_grad / scale, c["rot_grad"] / scale, atol=1e-9)
        np.testing.assert_allclose(fit.eigvals, c["eigvals"], atol=1e-13)
        np.testing.assert_allclose(fit.rot, c["rot"], atol=1e-9)
        if c["kind"] not in ("same", "rotated"):
            np.testing.assert_allclose(fit.quat, c["quat"], atol=1e-10)


def test_kearsley_fit_errors_and_degenerate_case(golden, cuda_device):
    g = golden("misc.npz")
    x, a = G.Structure(g["deg_x"]), G.Structure(g["deg_a"])
    with pytest.raises(errors.DegenerateFitError):
        G.kearsley_fit(x, a, with_derivatives=True)
    np.testing.assert_allclose(G.kearsley_fit(x, a).eigvals, g["deg_eigvals"], atol=1e-14)
    with pytest.raises(errors.InvalidStructureError):
        G.kearsley_fit(G.Structure(np.zeros((3, 3)) + np.arange(3)[:, None]), x)


def test_rotation_derivative_check(golden, cuda_device):
    g = golden("misc.npz")
    v = G.rotation_derivative_check(G.Structure(g["check_x"]), G.Structure(g["check_a"]))
    assert v < 1e-5
    assert abs(v - float(g["check_value"])) < 1e-7


def test_jacobi_eigh_matches_reference(golden, cuda_device):
    g = golden("jacobi.npz")
    for m, v, vec in list(zip(g["mats"], g["vals"], g["vecs"]))[:16]:
        w, u = G.jacobi_eigh(m)
        s = max(1.0, np.abs(m).max())
        np.testing.assert_allclose(w / s, v / s, atol=1e-13)
        np.testing.assert_allclose(u, vec, atol=1e-9)
    with pytest.raises(ValueError):
        G.jacobi_eigh(np.array([[1.0, 2.0], [0.0, 1.0]]))


def test_jacobi_eigh_general_n_matches_reference(golden, cuda_device):
    """geometry.jacobi_eigh for n != 4 and custom tol / max_sweeps (the general-n device
    kernel) against the reference's own outputs, RuntimeError where the reference raised."""
    g = golden("jacobi_n.npz")
    o1 = o2 = 0
    for n, tol, ms, ok in zip(g["sizes"], g["tols"], g["sweeps"], g["conv"]):
        n, tol, ms = int(n), float(tol), int(ms)
        m = g["mats"][o2:o2 + n * n].reshape(n, n)
        v, u = g["vals"][o1:o1 + n], g["vecs"][o2:o2 + n * n].reshape(n, n)
        o1, o2 = o1 + n, o2 + n * n
        if not ok:
            with pytest.raises(RuntimeError):
                G.jacobi_eigh(m, tol=tol, max_sweeps=ms)
            continue
        w, vec = G.jacobi_eigh(m, tol=tol, max_sweeps=ms)
        scale = max(1.0, np.abs(m).max())
        np.testing.assert_allclose(w / scale, v / scale, atol=1e-12)
        np.testing.assert_allclose(vec, u, atol=1e-8)


def test_exact_distance_vs_oracle(cuda_device):
    rng = np.random.default_rng(10)
    n = 6
    w, wa = rng.uniform(0.1, 1, n), rng.uniform(0.1, 1, n)
    x = G.Structure(rng.normal(scale=0.3, size=(n, 3)), w, wa)
    a = G.Structure(rng.normal(scale=0.3, size=(n, 3)), w, wa).center()
    res = msd.exact_distance(x, a)
    wn, wan = x.disp_weights, x.align_weights
    v, g, _ = O.exact_distance(O.center(x.coords, wan), a.coords, wn, wan)
    assert res.exact and abs(res.value - v) <= 1e-12
    np.testing.assert_allclose(res.grad, g, atol=1e-10 * np.abs(g).max())
    # identity and rigid-motion invariance
    same = msd.exact_distance(a, a)
    assert abs(same.value) < 1e-10 and np.abs(same.grad).max() < 1e-10
    q = synth.random_rotations(rng, 1)[0]
    moved = G.Structure(a.coords @ q.T + 0.7, w, wa)
    assert abs(msd.exact_distance(moved, a).value) < 1e-10


def test_close_structure_steps_vs_oracle(golden, cuda_device):
    g = golden("close.npz")
    frames, lms, eps = g["frames"], g["landmarks"], float(g["eps"])
    lam = 100.0
    ref = colvar.ReferenceSet([G.Structure(a).center() for a in lms], lam=lam)
    state = msd.CloseStructureState(epsilon=eps)
    orc = O.close_structure_replay(frames, lms, lam, eps)
    for t in range(frames.shape[0]):
        state, results = msd.step_close_structure(G.Structure(frames[t]), state, ref)
        vals = np.array([r.value for r in results])
        assert all(r.exact for r in results) == bool(orc["refresh"][t])
        np.testing.assert_allclose(vals, orc["D"][t], rtol=1e-9, atol=1e-12)
        cv = colvar.property_map(list(enumerate(results)), ref)
        assert abs(cv.value - orc["s"][t]) <= 1e-6 * max(1, abs(orc["s"][t]))
        assert abs(cv.z - orc["z"][t]) <= max(1e-6 * abs(orc["z"][t]), 1e-9)
        sc = np.abs(orc["ds"][t]).max()
        np.testing.assert_allclose(cv.grad, orc["ds"][t], atol=1e-5 * sc)
        np.testing.assert_allclose(cv.zgrad, orc["dz"][t], atol=1e-5 * np.abs(orc["dz"][t]).max())
        for r in results:
            assert np.abs(r.grad.sum(axis=0)).max() < 1e-8
    c = orc["counters"]
    assert state.reassign_count == c["reassign_count"]
    assert state.expensive_count == c["expensive_count"] == frames.shape[0] + state.reassign_count * len(lms)
    assert state.cheap_count == c["cheap_count"]


def test_approx_distance_equals_exact_after_reassignment(cuda_device):
    wl = synth.config0(seed=12, T=3, L=4, N=10)
    ref = colvar.ReferenceSet([G.Structure(a).center() for a in wl.landmarks], lam=wl.lam)
    state = msd.CloseStructureState(epsilon=1.0)
    x = G.Structure(wl.frames[0])
    state, exact = msd.step_close_structure(x, state, ref)
    state, approx = msd.step_close_structure(x, state, ref)  # D(x, y) = 0 <= eps: approximate
    assert not approx[0].exact
    for e, a in zip(exact, approx):
        assert abs(e.value - a.value) < 1e-12
    r = msd.approx_distance(x, 2, state, ref)
    assert abs(r.value - exact[2].value) < 1e-12


def test_approx_distance_right_after_a_single_reassigning_step(cuda_device):
    """after a refresh the state's x<->y fit is x against its own close
    structure (R_xy = I), so approx_distance equals the exact distance at once --
    on the first step and on a later refresh (where a stale fit to the old y
    would otherwise be combined with the new saved rotations)."""
    wl = synth.config0(seed=13, T=3, L=5, N=12)
    ref = colvar.ReferenceSet([G.Structure(a).center() for a in wl.landmarks], lam=wl.lam)
    state = msd.CloseStructureState(epsilon=1e-12)  # every distinct frame reassigns
    for t in range(3):
        x = G.Structure(wl.frames[t])
        state, exact = msd.step_close_structure(x, state, ref)
        assert all(r.exact for r in exact) and state.reassign_count == t + 1
        for i in (0, 3):
            r = msd.approx_distance(x, i, state, ref)
            assert abs(r.value - exact[i].value) < 1e-12
            np.testing.assert_allclose(r.grad, exact[i].grad, atol=1e-9 * max(1.0, np.abs(exact[i].grad).max()))


def test_property_map_kats(cuda_device):
    a = G.Structure(np.random.default_rng(0).normal(size=(4, 3)))
    ref1 = colvar.ReferenceSet([a], lam=3.0, properties=[7.0])
    r = msd.DistanceResult(0.4, np.ones((4, 3)), True)
    cv = colvar.property_map([(0, r)], ref1)
    assert cv.value == 7.0 and np.abs(cv.grad).max() == 0.0
    ref2 = colvar.ReferenceSet([a, a], lam=3.0, properties=[1.0, 2.0])
    cv = colvar.property_map([(0, msd.DistanceResult(0.2, None, True)), (1, msd.DistanceResult(0.2, None, True))],
                             ref2)
    assert abs(cv.value - 1.5) < 1e-15
    with pytest.raises(errors.EmptyActiveSetError):
        colvar.property_map([], ref2)
