"""Metadynamics bias / force (SPEC [MODULE] metadynamics, PAPER Eq. 1):
oracle pinned to the SPEC examples and properties; device kernels against the oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle as O


def test_oracle_mtd_spec_examples():
    V, dV = O.mtd_bias_direct([[0.3]], np.zeros((0, 1)), np.zeros((0, 1)), [])   # empty store
    assert V[0] == 0.0 and dV[0, 0] == 0.0
    V, _ = O.mtd_bias_direct([[0.0]], [[0.0]], [[0.2]], [1.7])                  # deposit at 0, query at 0
    assert V[0] == pytest.approx(1.7, rel=1e-15)
    V, _ = O.mtd_bias_direct([[0.2]], [[0.0]], [[0.2]], [1.7])                  # query at one sigma
    assert V[0] == pytest.approx(1.7 * np.exp(-0.5), rel=1e-14)
    _, dV = O.mtd_bias_direct([[0.4, -0.1]], [[0.4, -0.1]], [[0.2, 0.3]], [2.0])  # peak is stationary
    assert np.all(dV == 0.0)
    # product structure over CVs (<= 1e-12)
    v2, _ = O.mtd_bias_direct([[0.1, 0.25]], [[0.0, 0.0]], [[0.2, 0.3]], [1.0])
    v0, _ = O.mtd_bias_direct([[0.1]], [[0.0]], [[0.2]], [1.0])
    v1, _ = O.mtd_bias_direct([[0.25]], [[0.0]], [[0.3]], [1.0])
    assert abs(v2[0] - v0[0] * v1[0]) <= 1e-12


def test_oracle_mtd_finite_differences_and_grid():
    rng = np.random.default_rng(3)
    c = rng.uniform(-0.8, 0.8, (40, 2))
    sg = np.tile([0.15, 0.2], (40, 1))
    h = rng.uniform(0.5, 1.5, 40)
    x = rng.uniform(-0.7, 0.7, (25, 2))
    V, dV = O.mtd_bias_direct(x, c, sg, h)
    for i in range(2):
        e = np.zeros(2)
        e[i] = 1e-6
        fd = (O.mtd_bias_direct(x + e, c, sg, h)[0] - O.mtd_bias_direct(x - e, c, sg, h)[0]) / 2e-6
        np.testing.assert_allclose(dV[:, i], fd, rtol=1e-6, atol=1e-9)
    g = O.mtd_grid_new([-1.0, -1.0], [1.0, 1.0], [200, 200])
    for k in range(40):
        O.mtd_grid_deposit(g, c[k], sg[k], h[k])
    Vg, dVg = O.mtd_grid_eval(g, x)
    assert np.max(np.abs(Vg - V)) < 1e-5 and np.max(np.abs(dVg - dV)) < 1e-3
    with pytest.raises(ValueError):
        O.mtd_grid_eval(g, [[1.5, 0.0]])


def _store(d, grid, cuda_device):
    from paper_1801_02362_b200.metadynamics import HillStore

    sig = [0.15, 0.2][:d]
    return HillStore(d, stride=5, height=1.2, sigma=sig, grid=grid, device=cuda_device)


@pytest.mark.gpu
@pytest.mark.parametrize("d", [1, 2, 3])
def test_device_direct_bias_matches_oracle(d, cuda_device):
    from paper_1801_02362_b200.metadynamics import HillStore

    rng = np.random.default_rng(d)
    sig = [0.15, 0.2, 0.25][:d]
    st = HillStore(d, stride=2, height=0.9, sigma=sig, device=cuda_device)
    cs = rng.uniform(-0.8, 0.8, (300, d))
    for k, c in enumerate(cs):
        st.deposit(torch.tensor(c), 2 * k)
    x = rng.uniform(-0.9, 0.9, (1000, d))
    V, dV = st.bias(torch.tensor(x, device=cuda_device))
    Vr, dVr = O.mtd_bias_direct(x, cs, np.tile(sig, (300, 1)), np.full(300, 0.9))
    np.testing.assert_allclose(V.cpu().numpy(), Vr, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(dV.cpu().numpy(), dVr, rtol=1e-11, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("d", [1, 2])
def test_device_grid_matches_oracle_grid_and_direct(d, cuda_device):
    from paper_1801_02362_b200.errors import OutOfGridError

    rng = np.random.default_rng(10 + d)
    lo, hi, bins = [-1.0] * d, [1.0] * d, [160, 200][:d]
    st = _store(d, (lo, hi, bins), cuda_device)
    g = O.mtd_grid_new(lo, hi, bins)
    cs = rng.uniform(-0.8, 0.8, (60, d))
    for k, c in enumerate(cs):
        st.deposit(torch.tensor(c), 5 * k)
        O.mtd_grid_deposit(g, c, [0.15, 0.2][:d], 1.2)
    np.testing.assert_allclose(st.grid["val"].cpu().numpy(), g["val"], rtol=1e-12, atol=1e-13)
    x = rng.uniform(-0.95, 0.95, (777, d))
    V, dV = st.bias(torch.tensor(x, device=cuda_device))
    Vr, dVr = O.mtd_grid_eval(g, x)
    np.testing.assert_allclose(V.cpu().numpy(), Vr, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dV.cpu().numpy(), dVr, rtol=1e-10, atol=1e-10)
    # grid vs direct summation: within the interpolation tolerance of the bin width
    Vd, _ = st.bias(torch.tensor(x, device=cuda_device), use_grid=False)
    assert float((V - Vd).abs().max()) < 1e-4
    with pytest.raises(OutOfGridError):
        st.bias(torch.tensor([[1.5] * d], device=cuda_device))
    before = st.grid["val"].clone()
    with pytest.raises(OutOfGridError):
        st.deposit(torch.tensor([2.0] * d), 5 * 60)
    # a rejected deposit leaves the grid and the hill list unchanged
    assert torch.equal(st.grid["val"], before) and st.centers.shape[0] == 60


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_device_force_matches_oracle(dtype, cuda_device):
    rng = np.random.default_rng(5)
    st = _store(2, None, cuda_device)
    for k, c in enumerate(rng.uniform(-0.5, 0.5, (20, 2))):
        st.deposit(torch.tensor(c), 5 * k)
    T, n = 37, 301
    cv = torch.tensor(rng.uniform(-0.6, 0.6, (T, 2)), device=cuda_device)
    ds = torch.tensor(rng.normal(size=(T, n, 3)), device=cuda_device, dtype=dtype)
    dz = torch.tensor(rng.normal(size=(T, n, 3)), device=cuda_device, dtype=dtype)
    V, F = st.bias_and_force(cv, [ds, dz])
    _, dVr = O.mtd_bias_direct(cv.cpu().numpy(), st.centers.cpu().numpy(), st.sigmas.cpu().numpy(),
                               st.heights.cpu().numpy())
    Fr = O.mtd_force(dVr, [ds.double().cpu().numpy(), dz.double().cpu().numpy()])
    tol = 1e-6 if dtype == torch.float32 else 1e-12
    np.testing.assert_allclose(F.double().cpu().numpy(), Fr, rtol=tol, atol=tol)
    # a single hill at the current CV value: zero force (stationary Gaussian peak)
    one = _store(2, None, cuda_device).deposit(torch.tensor([0.1, -0.2]), 0)
    _, F1 = one.bias_and_force(torch.tensor([[0.1, -0.2]], device=cuda_device), [ds[:1], dz[:1]])
    assert float(F1.abs().max()) == 0.0


@pytest.mark.gpu
def test_hills_file_and_deposit_rules(tmp_path, cuda_device):
    from paper_1801_02362_b200.errors import ConfigError

    st = _store(2, None, cuda_device)
    st.deposit([0.1, 0.2], 0).deposit([0.3, -0.4], 5)
    with pytest.raises(ConfigError):
        st.deposit([0.0, 0.0], 7)          # step not a multiple of the stride
    p = tmp_path / "HILLS"
    st.write_hills(p)
    rows = [line.split() for line in p.read_text().splitlines()]
    assert rows[1][0] == "5" and float(rows[1][1]) == 0.3 and float(rows[1][5]) == 1.2 and len(rows[1]) == 6
