"""Pin the C restatement (CPU baseline) to the numpy oracle."""

import numpy as np

from oracle import c_oracle as C
from oracle import oracle as O
from paper_1801_02362_b200 import synth


def test_c_msd_matrix_matches_numpy_oracle():
    wl = synth.config0(seed=1, T=40, L=20, N=22)
    D, used = C.msd_matrix(wl.frames, wl.landmarks)
    assert used >= 1
    np.testing.assert_allclose(D, O.batch_msd_matrix(wl.frames, wl.landmarks), rtol=1e-11, atol=1e-15)


def test_c_path_cv_matches_numpy_oracle_weighted():
    rng = np.random.default_rng(2)
    n = 13
    w, wa = rng.uniform(0.1, 1, n), rng.uniform(0.1, 1, n)
    wl = synth.config0(seed=2, T=12, L=9, N=n)
    c = C.path_cv_exact(wl.frames, wl.landmarks, wl.lam, w=w, w_align=wa)
    o = O.path_cv_exact(wl.frames, wl.landmarks, wl.lam, w=w, w_align=wa)
    np.testing.assert_allclose(c["s"], o["s"], rtol=1e-10)
    np.testing.assert_allclose(c["z"], o["z"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(c["ds"], o["ds"], atol=1e-8 * np.abs(o["ds"]).max())
    np.testing.assert_allclose(c["dz"], o["dz"], atol=1e-8 * np.abs(o["dz"]).max())


def test_c_fits_match_reference_golden(golden):
    g = golden("pathcv0.npz")
    D, _ = C.msd_matrix(g["frames"], g["landmarks"])
    np.testing.assert_allclose(D, g["D"], rtol=1e-11, atol=1e-15)


def test_c_close_replay_matches_numpy_oracle(golden):
    g = golden("close.npz")
    c = C.close_replay(g["frames"], g["landmarks"], 100.0, float(g["eps"]))
    np.testing.assert_array_equal(c["refresh"], g["refresh"])
    o = O.close_structure_replay(g["frames"], g["landmarks"], 100.0, float(g["eps"]))
    np.testing.assert_allclose(c["s"], o["s"], rtol=1e-10)
    np.testing.assert_allclose(c["z"], o["z"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(c["ds"], o["ds"], atol=1e-8 * np.abs(o["ds"]).max())
    np.testing.assert_allclose(c["dz"], o["dz"], atol=1e-8 * np.abs(o["dz"]).max())
