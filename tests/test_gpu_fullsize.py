"""Parity at BASELINE.json's full sizes (GPU).

Where the CPU oracle cannot finish the whole config in seconds, the full-size
device run is checked through size-independent properties on every frame
(s within [min q, max q], z <= D_min of the window, translation-invariant
gradients) plus exact spot checks of sampled frames against the C oracle.
"""

import numpy as np
import pytest
import torch

from oracle import c_oracle as C
from paper_1801_02362_b200 import engine, synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_config1_fullsize_refresh_log_and_cv_vs_c_oracle(cuda_device):
    """All 20000 frames: identical refresh log; s, z within 1e-6; gradients of a subset."""
    wl = synth.config1()
    out = engine.close_structure_replay(wl.frames, wl.landmarks, wl.lam, wl.eps)
    ref = C.close_replay(wl.frames, wl.landmarks, wl.lam, wl.eps, grad=False)
    np.testing.assert_array_equal(out["refresh"].cpu().numpy(), ref["refresh"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)
    np.testing.assert_allclose(out["z"].cpu().numpy(), ref["z"], rtol=1e-6, atol=1e-9)
    d = out["dxy"].cpu().numpy()
    np.testing.assert_allclose(d[1:], ref["dxy"][1:], rtol=1e-6, atol=1e-9)
    sub = C.close_replay(wl.frames[:300], wl.landmarks, wl.lam, wl.eps)
    for key in ("ds", "dz"):
        got, r = out[key][:300].cpu().numpy(), sub[key]
        scale = np.abs(r).reshape(300, -1).max(axis=1)
        assert np.all(np.abs(got - r).reshape(300, -1).max(axis=1) <= 1e-5 * scale)


def test_config4_fullsize_properties_and_spot_checks(cuda_device):
    wl = synth.interp_config_device(4, 131072, 8192, 10000, 32, cuda_device)
    pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(cuda_device), wl.lam, wl.q)
    out = pcv.evaluate(wl.frames)
    s = out["s"].cpu().numpy()
    z = out["z"].cpu().numpy()
    assert np.isfinite(s).all() and np.isfinite(z).all()
    assert (s >= 0).all() and (s <= 8191).all()
    # z <= D_min (log-sum-exp of the window is >= the largest term)
    dmin = np.array([out["D_window"][t, : out["window_cnt"][t]].min().item() for t in range(0, 131072, 4099)])
    assert np.all(z[::4099] <= dmin + 1e-12)
    # uniform weights: the gradients carry no net translation
    for key in ("ds", "dz"):
        g = out[key][::997].double()
        net = g.sum(dim=1).abs().max().item()
        assert net <= 1e-5 * g.abs().max().item() * 10000 ** 0.5
    # exact spot checks against the C restatement of the reference (all 8192 landmarks)
    idx = [0, 65537, 131071]
    fr = wl.frames[idx].double().cpu().numpy()
    ref = C.path_cv_exact(fr, wl.landmarks.astype(np.float64), wl.lam)
    np.testing.assert_allclose(s[idx], ref["s"], rtol=1e-6)
    np.testing.assert_allclose(z[idx], ref["z"], rtol=1e-6, atol=1e-9)
    for key in ("ds", "dz"):
        got = out[key][idx].double().cpu().numpy()
        r = ref[key]
        scale = np.abs(r).reshape(3, -1).max(axis=1)
        assert np.all(np.abs(got - r).reshape(3, -1).max(axis=1) <= 1e-5 * scale)
