"""GPU tests of the int8 tensor-core (tcgen05 kind::i8, Ozaki digits) gradient
contraction (csrc/grad_i8.cu) against the fp64 DMMA kernel and the fp64 oracle,
and of the fused metadynamics bias force on the same kernel.

Tolerances (BASELINE.json north_star): gradients within 1e-5 of the per-frame
maximum vs the oracle; the int8 and DMMA contractions agree to 1e-6 of the
per-frame maximum (both are exact to ~1e-8 of the contraction's magnitude).
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1801_02362_b200 import engine, kernels as K, synth

pytestmark = pytest.mark.gpu


def _rel_rows(got, ref):
    got = got.reshape(got.shape[0], -1).astype(np.float64)
    ref = ref.reshape(ref.shape[0], -1).astype(np.float64)
    scale = np.abs(ref).max(axis=1)
    err = np.abs(got - ref).max(axis=1)
    return err / np.maximum(scale, 1e-300)


def test_landmark_digits_reconstruct_centred_coordinates(cuda_device):
    """mc_ldig_prep: sum_q d_q 2^(24-8q) 2^(eB-31) equals ac = lraw - lcen within 2^(eB-32)."""
    wl = synth.config4(seed=11, T=4, L=77, N=300)
    lm = torch.from_numpy(wl.landmarks).cuda()
    lcen = lm.double().mean(dim=1)
    ld = K.ldig_prep(lm, lcen)
    d4 = ld.dig.cpu().numpy().astype(np.int64)  # [npad, kpad / 32, 4, 32]
    dig = d4.transpose(2, 0, 1, 3).reshape(4, d4.shape[0], -1)  # [4, npad, kpad]
    eB = ld.eB.cpu().numpy()[:300]
    L, n = 77, 300
    X = dig[0] * 2 ** 24 + dig[1] * 2 ** 16 + dig[2] * 2 ** 8 + dig[3]  # [npad, kpad]
    rec = X[:n, :3 * L].astype(np.float64) * np.ldexp(1.0, eB - 31)[:, None]
    ac = (wl.landmarks.astype(np.float64) - lcen.cpu().numpy()[:, None, :])  # [L, n, 3]
    ref = ac.transpose(1, 0, 2).reshape(n, 3 * L)
    err = np.abs(rec - ref)
    assert np.all(err <= np.ldexp(1.0, eB - 32)[:, None] * (1 + 1e-12))
    assert np.all(np.abs(dig[0]) <= 127) and np.all(dig[:, n:, :] == 0) and np.all(dig[:, :, 3 * L:] == 0)
    # the leading digit of each atom's largest coordinate is near full scale
    assert np.all(np.abs(dig[0, :n, :3 * L]).max(axis=1) >= 63)


@pytest.mark.parametrize("T,L,N", [(96, 512, 600), (77, 300, 1000), (40, 2048, 2500)])
def test_i8_gradient_matches_dmma_and_oracle(T, L, N, cuda_device):
    """PathCVTC.evaluate with the int8 contraction == the fp64 DMMA contraction (1e-6 of the
    per-frame max), and both == the fp64 oracle (1e-5); ragged T, n % 128 != 0."""
    wl = synth.config4(seed=5, T=T, L=L, N=N)
    pcv = engine.PathCVTC(wl.landmarks, wl.lam)
    assert pcv.ldig is not None
    out = pcv.evaluate(wl.frames, out_dtype=torch.float64)
    ldig, pcv.ldig = pcv.ldig, None
    dm = pcv.evaluate(wl.frames, out_dtype=torch.float64)
    pcv.ldig = ldig
    ref = O.batch_path_cv_exact(wl.frames.astype(np.float64), wl.landmarks.astype(np.float64), wl.lam)
    for key in ("ds", "dz"):
        a, b = out[key].cpu().numpy(), dm[key].cpu().numpy()
        r_dm = _rel_rows(a, b)
        r_or = _rel_rows(a, ref[key])
        print(f"{key}: i8 vs dmma worst {r_dm.max():.2e}, i8 vs oracle worst {r_or.max():.2e}")
        assert r_dm.max() <= 1e-6
        assert r_or.max() <= 1e-5
    np.testing.assert_array_equal(out["s"].cpu().numpy(), dm["s"].cpu().numpy())


def test_i8_gradient_fp32_output_and_wide_groups(cuda_device):
    """fp32 outputs; a small lambda widens the significant windows past 117 landmarks, so
    part of the groups run on the streamed-A int8 kernel (mc_pathcv_grad_i8_wide) beside
    the resident-image one: still == DMMA."""
    wl = synth.config4(seed=6, T=64, L=1024, N=400)
    pcv = engine.PathCVTC(wl.landmarks, wl.lam * 0.02, window_cap=1024)
    out = pcv.evaluate(wl.frames)
    nsig = out["nsig"].cpu().numpy()
    assert nsig.max() > 117, "the case must exercise the wide-group fallback"
    ldig, pcv.ldig = pcv.ldig, None
    dm = pcv.evaluate(wl.frames)
    pcv.ldig = ldig
    for key in ("ds", "dz"):
        r = _rel_rows(out[key].cpu().numpy(), dm[key].cpu().numpy())
        assert r.max() <= 2e-6, f"{key}: {r.max():.2e}"


def test_i8_wide_groups_streamed_equal_dmma_fallback_and_force(cuda_device):
    """Very wide significant unions (several hundred landmarks: the A image is built in
    chunks of 12 k-steps and streamed with the B boxes): the streamed-A int8 gradient ==
    the DMMA fallback (1e-6 of the per-frame max); the fused force of wide 16-frame
    groups == -(V_s ds + V_z dz) without the two-output fallback."""
    wl = synth.config4(seed=12, T=72, L=1024, N=512)
    pcv = engine.PathCVTC(wl.landmarks, wl.lam * 0.004, window_cap=1024)
    out = pcv.evaluate(wl.frames, out_dtype=torch.float64)
    nsig = out["nsig"].cpu().numpy()
    assert nsig.max() > 400, nsig.max()
    saved = K.GRAD_I8_WIDE
    try:
        K.GRAD_I8_WIDE = False
        fb = pcv.evaluate(wl.frames, out_dtype=torch.float64)
    finally:
        K.GRAD_I8_WIDE = saved
    for key in ("ds", "dz"):
        r = _rel_rows(out[key].cpu().numpy(), fb[key].cpu().numpy())
        assert r.max() <= 1e-6, f"{key}: {r.max():.2e}"
    rng = np.random.default_rng(5)
    dV = torch.from_numpy(rng.normal(size=(72, 2))).cuda()
    of = pcv.evaluate(wl.frames, grad=False, out_dtype=torch.float64, dV=dV)
    ref = -(dV[:, 0, None, None] * out["ds"] + dV[:, 1, None, None] * out["dz"]).cpu().numpy()
    r = _rel_rows(of["force"].cpu().numpy(), ref)
    assert r.max() <= 1e-6, f"force: {r.max():.2e}"


def test_fused_bias_force_equals_contracted_gradients(cuda_device):
    """F = -(V_s ds + V_z dz) from one tensor-core contraction == the same combination of
    the separately computed gradients (1e-6 of the per-frame max)."""
    wl = synth.config4(seed=8, T=50, L=512, N=800)
    pcv = engine.PathCVTC(wl.landmarks, wl.lam)
    rng = np.random.default_rng(3)
    dV = torch.from_numpy(rng.normal(size=(50, 2))).cuda()
    out = pcv.evaluate(wl.frames, out_dtype=torch.float64, dV=dV)
    F = out["force"].cpu().numpy()
    ref = -(dV[:, 0, None, None] * out["ds"] + dV[:, 1, None, None] * out["dz"]).cpu().numpy()
    r = _rel_rows(F, ref)
    assert r.max() <= 1e-6, f"{r.max():.2e}"
    # zero net force (translation invariance): each atom's force is exact to ~1e-8 of the
    # frame's largest component, so the sum over the atoms vanishes to within the 1e-5
    # gradient tolerance (the fp64 DMMA sum to ~1e-14)
    assert np.abs(F.sum(axis=1)).max() <= 1e-5 * np.abs(F).max()


@pytest.mark.parametrize("T,L,N", [(96, 512, 600), (77, 300, 1000), (40, 2048, 2500)])
def test_i8_refits_match_dmma_refits_and_oracle(T, L, N, cuda_device):
    """Exact window refits on the int8 tensor cores (mc_refine_i8) == the fp64 DMMA refits:
    every window MSD within 1e-9 absolute + 1e-12 relative, and == the fp64 oracle's MSDs
    (1e-6 relative or 1e-9 absolute); s and z == the oracle (1e-6)."""
    wl = synth.config4(seed=9, T=T, L=L, N=N)
    pcv = engine.PathCVTC(wl.landmarks, wl.lam)
    assert pcv.rdl is not None
    a = pcv.evaluate(wl.frames, out_dtype=torch.float64)
    rdl, pcv.rdl = pcv.rdl, None
    b = pcv.evaluate(wl.frames, out_dtype=torch.float64)
    pcv.rdl = rdl
    np.testing.assert_array_equal(a["window_cnt"].cpu().numpy(), b["window_cnt"].cpu().numpy())
    cnt, lo = a["window_cnt"].cpu().numpy(), a["window_lo"].cpu().numpy()
    Da, Db = a["D_window"].cpu().numpy(), b["D_window"].cpu().numpy()
    ref = O.batch_msd_matrix(wl.frames.astype(np.float64), wl.landmarks.astype(np.float64))
    worst = 0.0
    for t in range(T):
        x, y = Da[t, :cnt[t]], Db[t, :cnt[t]]
        r = ref[t, lo[t]:lo[t] + cnt[t]]
        assert np.all(np.abs(x - y) <= 1e-9 + 1e-12 * np.abs(y)), np.abs(x - y).max()
        assert np.all(np.abs(x - r) <= np.maximum(1e-6 * np.abs(r), 1e-9))
        worst = max(worst, float(np.abs(x - r).max()))
    print(f"T={T} L={L} N={N}: worst |D_i8 - D_oracle| {worst:.2e}")
    # the int8 refits are exact to ~1e-10 absolute on D (31-bit operand digits), which moves
    # s and z by ~lam 1e-10: far inside the 1e-6 tolerance against the oracle
    ds_ = np.abs(a["s"].cpu().numpy() - b["s"].cpu().numpy()).max()
    dz_ = np.abs(a["z"].cpu().numpy() - b["z"].cpu().numpy()).max()
    print(f"  s: max |i8 - dmma| {ds_:.2e}; z: {dz_:.2e}")
    np.testing.assert_allclose(a["s"].cpu().numpy(), b["s"].cpu().numpy(), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(a["z"].cpu().numpy(), b["z"].cpu().numpy(), rtol=1e-8, atol=1e-10)
    ref_cv = O.batch_path_cv_exact(wl.frames.astype(np.float64), wl.landmarks.astype(np.float64), wl.lam)
    np.testing.assert_allclose(a["s"].cpu().numpy(), ref_cv["s"], rtol=1e-6)
    np.testing.assert_allclose(a["z"].cpu().numpy(), ref_cv["z"], rtol=1e-6, atol=1e-9)


def test_i8_dense_refits_near_identical_pairs(cuda_device):
    """Dense exact matrix (config-2 path) on the int8 kernel: a landmark under a rigid motion
    as a frame gives D ~ 0 within 1e-9 absolute; every pair within 1e-6 relative or 1e-9
    absolute of the oracle."""
    wl = synth.config2(seed=5, T=70, L=90, N=1000)
    rng = np.random.default_rng(2)
    frames = wl.frames.copy()
    frames[:20] = synth.rigid_motion(rng, wl.landmarks[:20].astype(np.float64), dtype=np.float32)
    pcv = engine.PathCVTC(wl.landmarks, wl.lam)
    D = pcv.msd_matrix(frames).cpu().numpy().astype(np.float64)
    ref = O.batch_msd_matrix(frames.astype(np.float64), wl.landmarks.astype(np.float64))
    assert np.all(np.abs(D - ref) <= np.maximum(1e-6 * np.abs(ref), 1e-9 + 6e-8 * np.abs(ref)))
    d0 = np.abs(D[np.arange(20), np.arange(20)] - ref[np.arange(20), np.arange(20)])
    assert d0.max() <= 1e-9, d0.max()


def test_row_digit_exponents_from_k1s_equal_two_pass(cuda_device):
    """mc_row_digits with the exponents of the uniform-weight K1s (per-axis extrema of its
    first pass; one pass over the coordinates) == the two-pass row digits: identical
    exponents and digits, in a permuted order, with a translated and a rescaled frame."""
    wl = synth.config4(seed=13, T=200, L=64, N=1000)
    x = torch.from_numpy(wl.frames).cuda()
    x[7] += 30.0
    x[11] *= 1e-3
    n = x.shape[1]
    w = torch.full((n,), 1.0 / n, dtype=torch.float64, device=x.device)
    sp = K.center_split(x, w, w, weighted=False, fmt="f16", terms=1, wuni=1.0 / n)
    assert sp.dexp is not None
    perm = torch.randperm(200, device=x.device).to(torch.int32)
    a = K.row_digits(x, sp.centroid, None, perm=perm)
    b = K.row_digits(x, sp.centroid, None, perm=perm, ein=sp.dexp)
    assert torch.equal(a.e, b.e)
    assert torch.equal(a.dig, b.dig)
    # the digit-plane layout (the refits' frame operand) is the same digits transposed
    c = K.row_digits(x, sp.centroid, None, perm=perm, ein=sp.dexp, planes=True)
    R3, nks = a.dig.shape[0], a.dig.shape[1]
    assert torch.equal(c.e, a.e)
    assert torch.equal(c.dig.reshape(nks, 4, R3, 32), a.dig.permute(1, 2, 0, 3))


@pytest.mark.gpu
def test_row_digit_planes_chunked_kernel_equals_two_pass(cuda_device):
    """The shared-memory-staged plane kernel (exponents from the K1s, w = 1; several 1280-atom
    chunks with a partial last one, rows gathered through perm and fmap) writes exactly the
    digits of the two-pass kernel."""
    rng = np.random.default_rng(5)
    T, n = 37, 2692
    x = torch.from_numpy(rng.normal(size=(T, n, 3)).astype(np.float32)).cuda()
    x[3] += 12.5
    w = torch.full((n,), 1.0 / n, dtype=torch.float64, device=x.device)
    sp = K.center_split(x, w, w, weighted=False, fmt="f16", terms=1, wuni=1.0 / n)
    perm = torch.randperm(T, device=x.device).to(torch.int32)
    a = K.row_digits(x, sp.centroid, None, perm=perm)
    c = K.row_digits(x, sp.centroid, None, perm=perm, ein=sp.dexp, planes=True)
    R3, nks = a.dig.shape[0], a.dig.shape[1]
    assert nks > 80  # more than two chunks
    assert torch.equal(c.e, a.e)
    assert torch.equal(c.dig.reshape(nks, 4, R3, 32), a.dig.permute(1, 2, 0, 3))
    # frames stored in another order, read through fmap (sorted position -> raw row)
    fmap = torch.randperm(T, device=x.device).to(torch.int32)
    xs = torch.empty_like(x)
    xs[fmap.long()] = x
    d = K.row_digits(xs, sp.centroid, None, perm=perm, fmap=fmap, count=T, ein=sp.dexp, planes=True)
    assert torch.equal(d.dig, c.dig) and torch.equal(d.e, c.e)
