"""GPU parity: libmcb200 kernels vs the CPU oracle / reference golden vectors.

Tolerances (north_star): MSD, s, z within 1e-6 relative (1e-9 absolute for
near-identical pairs); gradients within 1e-5 relative; refresh decisions
identical frame by frame.  The fp64 path is far tighter than that, and the
asserts below say so explicitly where they are tighter.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1801_02362_b200 import engine, kernels as K, synth
from paper_1801_02362_b200.errors import InvalidStructureError

pytestmark = pytest.mark.gpu

MSD_RTOL, MSD_ATOL = 1e-6, 1e-9
GRAD_RTOL = 1e-5


def assert_msd(got, ref, rtol=MSD_RTOL, atol=MSD_ATOL):
    got = np.asarray(got)
    ref = np.asarray(ref)
    err = np.abs(got - ref)
    tol = np.maximum(rtol * np.abs(ref), atol)
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside tolerance; worst {err.max():.3e}"


def assert_grad(got, ref, rtol=GRAD_RTOL):
    got = np.asarray(got, dtype=float)
    ref = np.asarray(ref, dtype=float)
    # per-frame relative to that frame's largest gradient component
    scale = np.abs(ref).reshape(ref.shape[0], -1).max(axis=1)
    err = np.abs(got - ref).reshape(ref.shape[0], -1).max(axis=1)
    assert np.all(err <= rtol * np.maximum(scale, 1e-300)), f"worst rel {np.max(err / np.maximum(scale, 1e-300)):.3e}"


def _fits(golden):
    g = golden("fits.npz")
    for i in range(int(g["count"])):
        yield {k.split("_", 1)[1]: g[k] for k in g.files if k.startswith(f"{i}_")}


def test_fit_kernels_vs_reference_golden(golden, cuda_device):
    for c in _fits(golden):
        n = int(c["n"])
        w = torch.zeros(K.npad_for(n), dtype=torch.float64, device=cuda_device)
        w[:n] = torch.from_numpy(c["w"])
        x = torch.from_numpy(c["xc"])[None].to(cuda_device)
        a = torch.from_numpy(c["ac"])[None].to(cuda_device)
        xc = K.center(x, None, w, recenter=False)
        ac = K.center(a, None, w, recenter=False)
        S = K.cov_pairs(xc.planes, ac.planes, None, None, xc.npad, w)
        eig, quat, rot, flags = K.fit_full(S, xc.g, ac.g)
        eig = eig.cpu().numpy()[0]
        np.testing.assert_allclose(eig[:4], c["eigvals"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(rot.cpu().numpy()[0].reshape(3, 3), c["rot"], atol=1e-9)
        if c["kind"] not in ("same", "rotated"):
            np.testing.assert_allclose(quat.cpu().numpy()[0], c["quat"], atol=1e-10)
        # fast path (Newton + adjugate)
        D, R, Q, fl = K.fit_dense(S.reshape(1, 1, 9), xc.g, ac.g, want_quat=True)
        assert_msd(D.cpu().numpy()[0, 0], c["eigvals"][0], rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(R.cpu().numpy()[0, 0].reshape(3, 3), c["rot"], atol=1e-7)
        if not bool(c["degenerate"]):
            assert not (int(flags.item()) & 1)
            rg = K.rot_grad(xc.planes, ac.planes, n, xc.npad, w, torch.from_numpy(eig[None]).to(cuda_device))
            ref = c["rot_grad"]
            scale = max(1.0, np.abs(ref).max())
            np.testing.assert_allclose(rg.cpu().numpy()[0] / scale, ref / scale, atol=1e-9)


def test_jacobi4_vs_reference_golden(golden, cuda_device):
    g = golden("jacobi.npz")
    vals, vecs, flags = K.jacobi4(torch.from_numpy(g["mats"].reshape(-1, 16)).to(cuda_device))
    scale = np.maximum(1.0, np.abs(g["mats"]).max(axis=(1, 2)))[:, None]
    np.testing.assert_allclose(vals.cpu().numpy() / scale, g["vals"] / scale, atol=1e-13)
    np.testing.assert_allclose(vecs.cpu().numpy(), g["vecs"], atol=1e-9)
    assert int(flags.max()) == 0


def test_msd_matrix_config0_and_config1_slice(cuda_device):
    wl = synth.config0()
    D = engine.msd_matrix(torch.from_numpy(wl.frames).to(cuda_device), wl.landmarks).cpu().numpy()
    assert_msd(D, O.batch_msd_matrix(wl.frames, wl.landmarks))
    wl1 = synth.config1(T=300, L=120)
    D = engine.msd_matrix(wl1.frames, wl1.landmarks).cpu().numpy()
    assert_msd(D, O.batch_msd_matrix(wl1.frames, wl1.landmarks))


def test_msd_matrix_weights_and_fp32_inputs(cuda_device):
    rng = np.random.default_rng(3)
    n = 37
    w = rng.uniform(0.1, 1.0, n)
    wa = rng.uniform(0.1, 1.0, n)
    wl = synth.config0(seed=5, T=50, L=30, N=n)
    D = engine.msd_matrix(wl.frames, wl.landmarks, w=w, w_align=wa).cpu().numpy()
    assert_msd(D, O.batch_msd_matrix(wl.frames, wl.landmarks, w=w, w_align=wa))
    f32 = wl.frames.astype(np.float32)
    l32 = wl.landmarks.astype(np.float32)
    D = engine.msd_matrix(f32, l32).cpu().numpy()
    assert_msd(D, O.batch_msd_matrix(f32.astype(float), l32.astype(float)))


def test_path_cv_config0_full(cuda_device):
    wl = synth.config0()
    out = engine.path_cv(wl.frames, wl.landmarks, wl.lam)
    ref = O.batch_path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    assert_msd(out["D"].cpu().numpy(), ref["D"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(out["z"].cpu().numpy(), ref["z"], rtol=1e-6, atol=1e-9)
    assert_grad(out["ds"].cpu().numpy(), ref["ds"])
    assert_grad(out["dz"].cpu().numpy(), ref["dz"])


def test_path_cv_vs_per_pair_oracle_with_rot_term(golden, cuda_device):
    """Against the literal Eq. 4 oracle (dR term included) on reference-fit slices."""
    g = golden("pathcv0.npz")
    out = engine.path_cv(g["frames"], g["landmarks"], float(g["lam"]))
    ref = O.path_cv_exact(g["frames"], g["landmarks"], float(g["lam"]))
    assert_msd(out["D"].cpu().numpy(), g["D"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)
    assert_grad(out["ds"].cpu().numpy(), ref["ds"])
    assert_grad(out["dz"].cpu().numpy(), ref["dz"])


def test_path_cv_weighted(cuda_device):
    rng = np.random.default_rng(4)
    n = 9
    w = rng.uniform(0.1, 1.0, n)
    wa = rng.uniform(0.1, 1.0, n)
    wl = synth.config0(seed=6, T=6, L=8, N=n)
    out = engine.path_cv(wl.frames, wl.landmarks, wl.lam, w=w, w_align=wa)
    ref = O.path_cv_exact(wl.frames, wl.landmarks, wl.lam, w=w, w_align=wa)
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)
    np.testing.assert_allclose(out["z"].cpu().numpy(), ref["z"], rtol=1e-6, atol=1e-9)
    assert_grad(out["ds"].cpu().numpy(), ref["ds"])
    assert_grad(out["dz"].cpu().numpy(), ref["dz"])


def test_close_replay_vs_reference_run(golden, cuda_device):
    g = golden("close.npz")
    out = engine.close_structure_replay(g["frames"], g["landmarks"], 100.0, float(g["eps"]))
    np.testing.assert_array_equal(out["refresh"].cpu().numpy(), g["refresh"])
    assert_msd(out["dxy"].cpu().numpy(), g["dxy"])
    assert_msd(out["D"].cpu().numpy(), g["D"])


def test_close_replay_gradients_vs_oracle(cuda_device):
    g_wl = synth.config0(seed=8, T=40, L=10, N=12)
    # small eps so that both refresh and approximate frames occur
    frames = g_wl.frames.copy()
    rng = np.random.default_rng(1)
    base = frames[0] - frames[0].mean(0)
    for t in range(frames.shape[0]):
        frames[t] = base + np.cumsum(rng.normal(0, 0.002, size=(t + 1, 12, 3)), axis=0)[-1]
    frames = synth.rigid_motion(rng, frames)
    eps = 3e-4
    lam = 50.0
    ref = O.close_structure_replay(frames, g_wl.landmarks, lam, eps)
    assert 0 < ref["refresh"].sum() < len(ref["refresh"])
    out = engine.close_structure_replay(frames, g_wl.landmarks, lam, eps)
    np.testing.assert_array_equal(out["refresh"].cpu().numpy(), ref["refresh"])
    assert_msd(out["dxy"].cpu().numpy(), ref["dxy"])
    assert_msd(out["D"].cpu().numpy(), ref["D"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)
    np.testing.assert_allclose(out["z"].cpu().numpy(), ref["z"], rtol=1e-6, atol=1e-9)
    assert_grad(out["ds"].cpu().numpy(), ref["ds"])
    assert_grad(out["dz"].cpu().numpy(), ref["dz"])


def test_close_replay_config1_slice_decisions(cuda_device):
    wl = synth.config1(T=400, L=60)
    ref = O.close_structure_replay(wl.frames, wl.landmarks, wl.lam, wl.eps, grad=False)
    out = engine.close_structure_replay(wl.frames, wl.landmarks, wl.lam, wl.eps, grad=False)
    np.testing.assert_array_equal(out["refresh"].cpu().numpy(), ref["refresh"])
    assert_msd(out["dxy"].cpu().numpy(), ref["dxy"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)
    # and with a large eps, so most frames take the approximate path
    eps = 50 * wl.eps
    ref = O.close_structure_replay(wl.frames[:120], wl.landmarks, wl.lam, eps, grad=False)
    out = engine.close_structure_replay(wl.frames[:120], wl.landmarks, wl.lam, eps, grad=False)
    np.testing.assert_array_equal(out["refresh"].cpu().numpy(), ref["refresh"])
    assert ref["refresh"].sum() < 100
    assert_msd(out["D"].cpu().numpy(), ref["D"])
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"], rtol=1e-6)


def test_eps_zero_equals_exact(cuda_device):
    wl = synth.config0(seed=2, T=30, L=12, N=15)
    ex = engine.path_cv(wl.frames, wl.landmarks, wl.lam)
    cl = engine.close_structure_replay(wl.frames, wl.landmarks, wl.lam, 0.0)
    assert bool(cl["refresh"].all())
    np.testing.assert_allclose(cl["s"].cpu().numpy(), ex["s"].cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(cl["ds"].cpu().numpy(), ex["ds"].cpu().numpy(), atol=1e-14)


def test_config3_walkers_slice_vs_oracle(cuda_device):
    """Config-3 generator (device) at reduced size: per-walker close structure,
    refresh logs identical, s/z/gradients vs the per-walker oracle replay."""
    from paper_1801_02362_b200 import synth as S

    wl = S.walkers_device(3, 256, 40, 60, 48, cuda_device, walker_offset=5, walker_count=3)
    out = engine.close_structure_replay(wl.frames, wl.landmarks, wl.lam, wl.eps)
    fr = wl.frames.double().cpu().numpy()
    for k in range(3):
        ref = O.close_structure_replay(fr[k], wl.landmarks.astype(np.float64), wl.lam, wl.eps)
        sl = slice(k * 40, (k + 1) * 40)
        np.testing.assert_array_equal(out["refresh"].cpu().numpy()[sl], ref["refresh"])
        np.testing.assert_allclose(out["s"].cpu().numpy()[sl], ref["s"], rtol=1e-6)
        np.testing.assert_allclose(out["z"].cpu().numpy()[sl], ref["z"], rtol=1e-6, atol=1e-9)
        assert_grad(out["ds"].cpu().numpy()[sl], ref["ds"])
        assert_grad(out["dz"].cpu().numpy()[sl], ref["dz"])
    assert 0 < out["refresh"].sum() < 120


def test_cov_dmma_matches_cov_f64(cuda_device):
    """Dense covariances on the fp64 tensor cores (raw fp32 operands, RAW epilogue)
    = the fp64-plane CUDA-core contraction, to fp64 rounding."""
    from paper_1801_02362_b200 import synth as S

    wl = S.walkers_device(4, 8, 6, 64, 40, cuda_device)
    fr = wl.frames.reshape(-1, 64, 3).contiguous()
    pcv = engine.PathCV(torch.from_numpy(wl.landmarks).to(cuda_device), wl.lam, wl.q)
    assert pcv.lraw is not None
    c = K.center(fr, pcv.wa, pcv.w)
    s_tc = K.cov_dmma(fr, c, pcv.lraw, pcv.lm, pcv.w, pcv.wuni).cpu().numpy()
    s_ref = K.cov_dense(c, pcv.lm).cpu().numpy()
    scale = np.abs(s_ref).max()
    assert np.abs(s_tc - s_ref).max() <= 1e-13 * scale


def test_close_replay_dmma_path_equals_fp64_path(cuda_device):
    """Config-3 shapes (fp32, N % 4 == 0): the DMMA close-structure path (dense S on
    DMMA, gradient contraction on DMMA + the Eq. 6 correction) against the
    fp64-plane CUDA-core path: identical refresh log, s/z to 1e-10 (fp64 summation
    order; the weights amplify it by lam * |dD|), gradients to fp32 output rounding."""
    from paper_1801_02362_b200 import synth as S

    wl = S.walkers_device(5, 64, 60, 96, 120, cuda_device, walker_offset=3, walker_count=4)
    lm = torch.from_numpy(wl.landmarks).to(cuda_device)
    a = engine.PathCV(lm, wl.lam, wl.q)
    assert a.lraw is not None
    saved = engine.CLOSE_DMMA, engine.CLOSE_PRUNE
    try:
        engine.CLOSE_DMMA = False
        b = engine.PathCV(lm, wl.lam, wl.q)
        engine.CLOSE_DMMA, engine.CLOSE_PRUNE = saved[0], False  # the dense DMMA path
        oa = a.close_replay(wl.frames, wl.eps, grad=True)
    finally:
        engine.CLOSE_DMMA, engine.CLOSE_PRUNE = saved
    assert b.lraw is None
    ob = b.close_replay(wl.frames, wl.eps, grad=True)
    np.testing.assert_array_equal(oa["refresh"].cpu().numpy(), ob["refresh"].cpu().numpy())
    assert 0 < int(oa["refresh"].sum()) < oa["refresh"].numel()
    np.testing.assert_allclose(oa["s"].cpu().numpy(), ob["s"].cpu().numpy(), rtol=1e-10)
    np.testing.assert_allclose(oa["z"].cpu().numpy(), ob["z"].cpu().numpy(), rtol=1e-10, atol=1e-15)
    for key in ("ds", "dz"):
        assert_grad(oa[key].cpu().numpy(), ob[key].cpu().numpy(), rtol=1e-6)


@pytest.mark.parametrize("seed,W,steps,n,L", [(5, 4, 60, 96, 120), (7, 3, 80, 200, 400), (9, 2, 50, 64, 1000)])
def test_close_replay_pruned_equals_dense(seed, W, steps, n, L, cuda_device):
    """Pruned close-structure replay (screened lifetime windows of the refresh frames,
    covariances and refresh fits on the int8 tensor cores) = the dense replay (every
    landmark's covariance on DMMA): identical refresh log, s and z to 2e-7 relative / 1e-10
    absolute (the int8 digits are exact to 2^-31 of each row's maximum: ~1e-10 on D, against
    fp64 DMMA), gradients to 1e-6 of the per-frame maximum; every frame's significant
    landmarks inside its window."""
    from paper_1801_02362_b200 import synth as S

    wl = S.walkers_device(seed, 64, steps, n, L, cuda_device, walker_offset=1, walker_count=W)
    lm = torch.from_numpy(wl.landmarks).to(cuda_device)
    pcv = engine.PathCV(lm, wl.lam, wl.q)
    assert pcv._close_prunable(wl.frames.reshape(-1, n, 3))
    op = pcv.close_replay(wl.frames, wl.eps, grad=True)
    assert "window_cnt" in op
    saved = engine.CLOSE_PRUNE
    try:
        engine.CLOSE_PRUNE = False
        od = pcv.close_replay(wl.frames, wl.eps, grad=True)
    finally:
        engine.CLOSE_PRUNE = saved
    assert "window_cnt" not in od
    np.testing.assert_array_equal(op["refresh"].cpu().numpy(), od["refresh"].cpu().numpy())
    assert 0 < int(op["refresh"].sum()) < op["refresh"].numel()
    np.testing.assert_allclose(op["s"].cpu().numpy(), od["s"].cpu().numpy(), rtol=2e-7, atol=1e-10)
    np.testing.assert_allclose(op["z"].cpu().numpy(), od["z"].cpu().numpy(), rtol=2e-7, atol=1e-10)
    for key in ("ds", "dz"):
        assert_grad(op[key].cpu().numpy(), od[key].cpu().numpy(), rtol=1e-6)
    # the dense distances of every landmark within the cutoff lie in the window
    D = od["D"].cpu().numpy()
    lo, cnt = op["window_lo"].cpu().numpy(), op["window_cnt"].cpu().numpy()
    sig = wl.lam * (D - D.min(axis=1, keepdims=True)) <= pcv.cutoff
    idx = np.arange(D.shape[1])[None, :]
    inside = (idx >= lo[:, None]) & (idx < (lo + cnt)[:, None])
    assert np.all(inside[sig])


def test_cuda_graph_replay_equals_eager(cuda_device):
    """PathCVGraph (config-0 shape): the replayed pipeline gives the eager evaluate()'s
    s, z and gradients bit for bit, for several inputs; errors surface through check()."""
    wl = synth.config0()
    pcv = engine.PathCV(torch.from_numpy(wl.landmarks).to(cuda_device), wl.lam, wl.q)
    g = pcv.graph(wl.frames.shape[0])
    for k in range(3):
        fr = torch.from_numpy(wl.frames + 0.01 * k).to(cuda_device)
        out = g.evaluate(fr)
        g.check()
        ref = pcv.evaluate(fr, grad=True, cap=pcv.L)
        for key in ("s", "z", "ds", "dz"):
            assert torch.equal(out[key], ref[key]), key
    bad = torch.from_numpy(wl.frames.copy()).to(cuda_device)
    bad[5, 3, 1] = float("nan")
    g.evaluate(bad)
    with pytest.raises(InvalidStructureError):
        g.check()


@pytest.mark.parametrize("T,L,n", [(70, 45, 50), (33, 97, 304), (5, 3, 22)])
def test_cov_f64_dmma_vs_numpy(T, L, n, cuda_device):
    """fp64-plane covariance on the fp64 tensor cores (cov_dmma_f64_kernel, the default for
    fp64 inputs) = the fp64 numpy contraction of the same planes, to fp64 rounding; ragged
    T, L (not multiples of the 32 x 32 tile) and padded atom counts."""
    rng = np.random.default_rng(T + L + n)
    x = torch.from_numpy(rng.normal(0, 0.5, size=(T, n, 3))).to(cuda_device)
    a = torch.from_numpy(rng.normal(0, 0.5, size=(L, n, 3))).to(cuda_device)
    w = torch.from_numpy(rng.uniform(0.5, 1.5, size=n) / n).to(cuda_device)
    wp = torch.zeros(K.npad_for(n), dtype=torch.float64, device=cuda_device)
    wp[:n] = w
    fx = K.center(x, wp, wp)
    fa = K.center(a, wp, wp, weighted=True)
    S = K.cov_dense(fx, fa).cpu().numpy()
    xp, ap = fx.planes.cpu().numpy(), fa.wplanes.cpu().numpy()
    ref = np.einsum("tbj,lgj->tlbg", xp, ap).reshape(T, L, 9)
    assert np.abs(S - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("factor", [0.5, 4.0, 30.0])
def test_close_scan_parallel_chain_equals_serial_walk(factor, cuda_device):
    """The pointer-doubling refresh chain (parallel pass of close_scan_kernel) gives the
    serial walk's refresh log, close-structure indices and D(x, y) exactly -- frequent
    refreshes (chain resolved in parallel) and rare ones (successor beyond the window:
    serial fallback with on-the-fly fits)."""
    import os

    rng = np.random.default_rng(int(factor * 10))
    wl = synth.config0(seed=9, T=4, L=12, N=16)
    steps = 300
    x = np.cumsum(rng.normal(0, 0.002, size=(steps, 16, 3)), axis=0) + wl.landmarks[3][None]
    frames = torch.from_numpy(x).to(cuda_device)
    pcv = engine.PathCV(torch.from_numpy(wl.landmarks).to(cuda_device), wl.lam)
    # eps = factor x the one-step MSD: refreshes every frame (0.5), every few frames (4,
    # inside the 8-frame window: resolved in parallel), or rarely (30: successors beyond
    # the window -> serial walk with on-the-fly fits)
    eps = factor * float(np.mean(np.sum((x[1:] - x[:-1]) ** 2, axis=(1, 2)) / 16))
    par = pcv.close_replay(frames, eps, grad=False)
    os.environ["MC_CLOSE_SCAN_SERIAL"] = "1"
    try:
        ser = pcv.close_replay(frames, eps, grad=False)
    finally:
        del os.environ["MC_CLOSE_SCAN_SERIAL"]
    for key in ("refresh", "dxy", "s", "z"):
        assert torch.equal(par[key], ser[key]), key
    n = int(par["refresh"].sum())
    print(f"eps = {factor} x step MSD: {n} refreshes in {steps}")
    assert (n > 0.9 * steps) if factor < 1 else (1 < n < steps)
