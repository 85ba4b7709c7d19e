"""Neighbour list (SPEC [MODULE] neighbourlist): oracle pinned to
the SPEC examples; device top-M selection and the neighbour-list replay against
the oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle as O


def test_oracle_neighbour_update_spec_examples():
    assert list(O.neighbour_update([0.5, 0.1, 0.3], 2)) == [1, 2]          # order statistics
    assert list(O.neighbour_update([0.2] * 6, 4)) == [0, 1, 2, 3]          # ties by lower index
    assert list(O.neighbour_update([0.9, 0.1, 0.5, 0.3], 4)) == [0, 1, 2, 3]  # M = N: all
    with pytest.raises(ValueError):
        O.neighbour_update([0.1, 0.2], 3)                                  # M > N: configuration error


def test_oracle_replay_full_list_equals_plain_replay():
    from paper_1801_02362_b200 import synth

    wl = synth.config1(T=12, L=10, N=16)
    a = O.close_structure_replay(wl.frames, wl.landmarks, wl.lam, wl.eps)
    b = O.close_structure_replay(wl.frames, wl.landmarks, wl.lam, wl.eps, neighbours=10, nl_stride=3)
    np.testing.assert_allclose(a["s"], b["s"], rtol=1e-13)
    np.testing.assert_allclose(a["z"], b["z"], rtol=1e-13)
    np.testing.assert_allclose(a["ds"], b["ds"], rtol=1e-12, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("L,M", [(1, 1), (7, 3), (500, 1), (500, 40), (2048, 2048), (8192, 64)])
def test_device_topm_matches_oracle(dtype, L, M, cuda_device):
    rng = np.random.default_rng(L * 31 + M)
    rows = 9
    D = rng.random((rows, L))
    D[::2] = np.round(D[::2] * 16) / 16  # many ties on even rows
    D[1, : min(L, 5)] = -1e-17           # tiny negative estimates order before zeros
    Dt = torch.tensor(D, dtype=dtype, device=cuda_device)
    from paper_1801_02362_b200 import kernels as K

    got = K.neighbour_topm(Dt, M).cpu().numpy()
    Dref = Dt.double().cpu().numpy()
    for r in range(rows):
        np.testing.assert_array_equal(got[r], O.neighbour_update(Dref[r], M))
    sel = torch.tensor([4, 0, 7], dtype=torch.int32)
    got2 = K.neighbour_topm(Dt, M, rows=sel).cpu().numpy()
    for k, r in enumerate([4, 0, 7]):
        np.testing.assert_array_equal(got2[k], O.neighbour_update(Dref[r], M))


@pytest.mark.gpu
def test_neighbour_list_class_semantics(cuda_device):
    from paper_1801_02362_b200.errors import ConfigError
    from paper_1801_02362_b200.neighbourlist import NeighbourList

    nl = NeighbourList(3, 2, stride=5, device=cuda_device)
    nl.maybe_update(0, torch.tensor([0.5, 0.1, 0.3]))
    assert nl.indices.cpu().tolist() == [1, 2] and nl.last_update_step == 0
    nl.maybe_update(3, torch.tensor([0.0, 0.9, 0.9]))  # not due: immutable between updates
    assert nl.indices.cpu().tolist() == [1, 2]
    nl.maybe_update(5, torch.tensor([0.0, 0.9, 0.9]))
    assert nl.indices.cpu().tolist() == [0, 1] and nl.last_update_step == 5
    off = NeighbourList(4, 2, stride=9, enabled=False, device=cuda_device)
    off.maybe_update(0, torch.tensor([0.4, 0.3, 0.2, 0.1]))
    assert off.indices.cpu().tolist() == [0, 1, 2, 3] and off.stride == 1
    with pytest.raises(ConfigError):
        NeighbourList(3, 4, device=cuda_device)


@pytest.mark.gpu
@pytest.mark.parametrize("M,stride", [(4, 1), (6, 5), (20, 3)])
def test_replay_with_neighbour_list_matches_oracle(M, stride, cuda_device):
    from paper_1801_02362_b200 import engine, synth

    wl = synth.config1(T=30, L=20, N=22)
    eps = wl.eps * 3.0  # mix of refresh and approximated frames
    ref = O.close_structure_replay(wl.frames, wl.landmarks, wl.lam, eps, neighbours=M, nl_stride=stride)
    out = engine.PathCV(wl.landmarks, wl.lam).close_replay(wl.frames, eps, neighbours=M, nl_stride=stride)
    np.testing.assert_array_equal(out["refresh"].cpu().numpy(), ref["refresh"])
    np.testing.assert_array_equal(out["active"].cpu().numpy(), ref["active"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)
    np.testing.assert_allclose(out["z"].cpu().numpy(), ref["z"], rtol=1e-6, atol=1e-9)
    for key in ("ds", "dz"):
        got, r = out[key].cpu().numpy(), ref[key]
        scale = np.abs(r).reshape(r.shape[0], -1).max(axis=1) + 1e-300
        err = np.abs(got - r).reshape(r.shape[0], -1).max(axis=1)
        assert np.all(err <= 1e-5 * scale), f"{key}: worst rel {np.max(err / scale):.3e}"


def _grad_close(got, r, rtol=1e-5):
    scale = np.abs(r).reshape(r.shape[0], -1).max(axis=1) + 1e-300
    err = np.abs(got - r).reshape(r.shape[0], -1).max(axis=1)
    assert np.all(err <= rtol * scale), f"worst rel {np.max(err / scale):.3e}"


@pytest.mark.gpu
@pytest.mark.parametrize("M,stride", [(5, 1), (12, 4)])
def test_tensor_core_neighbour_list_matches_oracle(M, stride, cuda_device):
    """PathCVTC.evaluate_nl (fp32 frames; certified top-M of the update frames from the
    one-term screen + exact int8 refits of the candidates) == the oracle's exact-mode
    replay with the same neighbour list (eps = 0: every frame exact): identical active
    sets, s / z within 1e-6, gradients within 1e-5."""
    from paper_1801_02362_b200 import engine, synth

    wl = synth.config4(seed=21, T=12, L=60, N=40)
    ref = O.close_structure_replay(wl.frames.astype(np.float64), wl.landmarks.astype(np.float64), wl.lam, 0.0,
                                   neighbours=M, nl_stride=stride)
    assert ref["refresh"].all()
    out = engine.PathCVTC(wl.landmarks, wl.lam).evaluate_nl(wl.frames, M, nl_stride=stride, out_dtype=torch.float64)
    np.testing.assert_array_equal(out["active"].cpu().numpy(), ref["active"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)
    np.testing.assert_allclose(out["z"].cpu().numpy(), ref["z"], rtol=1e-6, atol=1e-9)
    for key in ("ds", "dz"):
        _grad_close(out[key].cpu().numpy(), ref[key])


@pytest.mark.gpu
@pytest.mark.parametrize("M,stride,walkers", [(16, 1, 1), (40, 5, 2), (300, 1, 1)])
def test_tensor_core_neighbour_list_matches_fp64_engine(M, stride, walkers, cuda_device):
    """At larger shapes (L = 1024, N = 400, window-limited screen): evaluate_nl == the fp64
    engine's exact-mode close replay with the neighbour list (close_replay(eps=0,
    neighbours=M), itself pinned to the oracle above): identical active sets, s / z 1e-6,
    gradients 1e-5; with M larger than the significant set the result equals the
    list-free evaluate."""
    from paper_1801_02362_b200 import engine, synth

    wl = synth.config4(seed=22, T=48, L=1024, N=400)
    fr = torch.from_numpy(wl.frames).to(cuda_device)
    if walkers > 1:
        fr = fr.reshape(walkers, -1, 400, 3)
    tc = engine.PathCVTC(wl.landmarks, wl.lam)
    out = tc.evaluate_nl(fr, M, nl_stride=stride, out_dtype=torch.float64)
    saved = engine.CLOSE_PRUNE
    try:
        engine.CLOSE_PRUNE = False  # dense exact distances: the list from every landmark
        ref = engine.PathCV(wl.landmarks, wl.lam).close_replay(fr.double(), 0.0, walkers=1, neighbours=M,
                                                               nl_stride=stride)
    finally:
        engine.CLOSE_PRUNE = saved
    assert bool(ref["refresh"].all())
    np.testing.assert_array_equal(out["active"].cpu().numpy(), ref["active"].cpu().numpy())
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"].cpu().numpy(), rtol=1e-6)
    np.testing.assert_allclose(out["z"].cpu().numpy(), ref["z"].cpu().numpy(), rtol=1e-6, atol=1e-9)
    for key in ("ds", "dz"):
        _grad_close(out[key].cpu().numpy(), ref[key].cpu().numpy())
    if M == 300:
        full = tc.evaluate(wl.frames, out_dtype=torch.float64)
        np.testing.assert_allclose(out["s"].cpu().numpy(), full["s"].cpu().numpy(), rtol=1e-9)
