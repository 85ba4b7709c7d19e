"""GPU tests of the landmark-sharded evaluation.

G shard engines run in one process on one GPU, driven in lock step by
``dist.drive_lockstep`` (the collectives computed locally with the same merge
arithmetic as ``dist.DistComm``; no rank waits on another's kernels).  The
merged s, z and the owner rows of ds, dz must equal the unsharded evaluate() on
the full landmark set, and that one the oracle.  A real one-rank NCCL group runs
the same generator through ``evaluate_sharded``.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import oracle as O
from paper_1801_02362_b200 import dist as D
from paper_1801_02362_b200 import engine, synth

pytestmark = pytest.mark.gpu


# sharded vs unsharded gradients: both contractions run on the int8 tensor cores, exact to
# ~3e-8 of the per-frame maximum, but each shard scales its own coefficient digits, so the
# two sums round differently: agreement to 1e-6 (the oracle tolerance is 1e-5)
SHARD_REL = 1e-6


def _rows_close(x, y, rel):
    """Per-frame max-norm comparison (the gradient tolerance of the north_star)."""
    x = x.reshape(x.shape[0], -1)
    y = y.reshape(y.shape[0], -1)
    scale = np.abs(y).max(axis=1)
    err = np.abs(x - y).max(axis=1)
    assert np.all(err <= rel * scale + 1e-300), float((err / scale).max())


def _sharded(wl, G, bounds=None, **kw):
    engs = [engine.PathCVTC(wl.landmarks, wl.lam, shard=(g, G, bounds), **kw) for g in range(G)]
    outs = D.drive_lockstep([e.sharded_steps(wl.frames, out_dtype=torch.float64) for e in engs])
    return engs, outs


@pytest.mark.parametrize("G,L", [(1, 1536), (2, 1536), (3, 1536), (4, 384)])
def test_landmark_sharded_matches_unsharded(G, L, cuda_device):
    wl = synth.config4(T=260, L=L, N=240)
    full = engine.PathCVTC(wl.landmarks, wl.lam)
    ref = full.evaluate(wl.frames, out_dtype=torch.float64)
    engs, outs = _sharded(wl, G)
    # pruning is on whenever a shard has >= 16 landmark tiles
    assert [e.prune for e in engs] == [(e.L + 47) // 48 >= 16 for e in engs]
    s_ref, z_ref = ref["s"].cpu().numpy(), ref["z"].cpu().numpy()
    owner = outs[0]["owner"].cpu().numpy()
    for g, o in enumerate(outs):
        # every shard holds the merged s, z (bitwise the same on all shards)
        np.testing.assert_array_equal(o["s"].cpu().numpy(), outs[0]["s"].cpu().numpy())
        np.testing.assert_allclose(o["s"].cpu().numpy(), s_ref, rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(o["z"].cpu().numpy(), z_ref, rtol=1e-9, atol=1e-12)
        mine = owner == g
        if mine.any():
            # a shard's significant set is taken against its own window minimum (>= the
            # global one): a superset of the unsharded set, the extra landmarks below
            # e^-cutoff weight (amplified ~1e3 by the cancellation in ds)
            for key in ("ds", "dz"):
                _rows_close(o[key].cpu().numpy()[mine], ref[key].cpu().numpy()[mine], SHARD_REL)
    # every frame has exactly one owner, and with G > 1 the windows are split: most
    # frames have an empty window on some shard (the global-minimum exchange)
    assert set(np.unique(owner)) <= set(range(G))
    if G > 1:
        active = torch.isfinite(outs[0]["z_parts"]).sum(0).cpu().numpy()
        assert active.min() >= 1 and (active < G).mean() > 0.5
        # the same windows split over the shards (up to the hull gaps at shard boundaries
        # and the unscanned margins of the banded screen)
        tot = sum(int(o["window_cnt"].sum().item()) for o in outs)
        rtot = int(ref["window_cnt"].sum().item())
        assert abs(tot - rtot) <= 0.05 * rtot, (tot, rtot)


def test_landmark_sharded_vs_oracle(cuda_device):
    wl = synth.config4(T=40, L=1536, N=240)
    _, outs = _sharded(wl, 2)
    ref = O.batch_path_cv_exact(wl.frames.astype(np.float64), wl.landmarks.astype(np.float64), wl.lam)
    owner = outs[0]["owner"].cpu().numpy()
    for g, o in enumerate(outs):
        np.testing.assert_allclose(o["s"].cpu().numpy(), ref["s"], rtol=1e-6)
        np.testing.assert_allclose(o["z"].cpu().numpy(), ref["z"], rtol=1e-6, atol=1e-9)
        mine = owner == g
        for key in ("ds", "dz"):
            _rows_close(o[key].cpu().numpy()[mine], ref[key][mine], 1e-5)


def test_work_balanced_landmark_shards(cuda_device):
    """Contiguous shards cut at equal window load (landmark_load + balanced_bounds): the
    same results as the unsharded evaluate, with uneven shard sizes."""
    wl = synth.config4(T=260, L=1536, N=240)
    full = engine.PathCVTC(wl.landmarks, wl.lam)
    load = full.landmark_load(wl.frames[:128])
    assert int(load.sum().item()) == int(full.evaluate(wl.frames[:128], grad=False)["window_cnt"].sum().item())
    b = D.balanced_bounds(load, 3)
    ref = full.evaluate(wl.frames, out_dtype=torch.float64)
    engs, outs = _sharded(wl, 3, bounds=b)
    assert [e.L for e in engs] == [b[1] - b[0], b[2] - b[1], b[3] - b[2]]
    owner = outs[0]["owner"].cpu().numpy()
    for g, o in enumerate(outs):
        np.testing.assert_allclose(o["s"].cpu().numpy(), ref["s"].cpu().numpy(), rtol=1e-9, atol=1e-12)
        mine = owner == g
        for key in ("ds", "dz"):
            _rows_close(o[key].cpu().numpy()[mine], ref[key].cpu().numpy()[mine], SHARD_REL)


def test_landmark_shard_window_overflow_retry(cuda_device):
    """A window wider than the capacity on any shard makes every shard retry."""
    wl = synth.config4(T=24, L=256, N=200)
    ref = engine.PathCVTC(wl.landmarks, wl.lam).evaluate(wl.frames, out_dtype=torch.float64)
    _, outs = _sharded(wl, 2, window_cap=4)
    np.testing.assert_allclose(outs[1]["s"].cpu().numpy(), ref["s"].cpu().numpy(), rtol=1e-9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_landmark_sharded_through_nccl_one_rank(cuda_device):
    """evaluate_sharded over a real NCCL process group (world size 1 on one GPU)."""
    wl = synth.config4(T=64, L=1536, N=240)
    init = not dist.is_initialized()
    if init:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=cuda_device)
    try:
        eng = engine.PathCVTC(wl.landmarks, wl.lam, shard=(0, 1))
        out = eng.evaluate_sharded(wl.frames, out_dtype=torch.float64)
        torch.cuda.synchronize()
    finally:
        if init:
            dist.destroy_process_group()
    ref = engine.PathCVTC(wl.landmarks, wl.lam).evaluate(wl.frames, out_dtype=torch.float64)
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"].cpu().numpy(), rtol=1e-12)
    assert bool((out["owner"] == 0).all())
    _rows_close(out["ds"].cpu().numpy(), ref["ds"].cpu().numpy(), SHARD_REL)


def _routed(wl, G, bounds, **kw):
    T = wl.frames.shape[0]
    engs = [engine.PathCVTC(wl.landmarks, wl.lam, shard=(g, G, bounds), route=True, **kw) for g in range(G)]
    gens = []
    for g, e in enumerate(engs):
        off, cnt = D.shard_range(T, g, G)
        gens.append(e.routed_steps(wl.frames[off:off + cnt], off, T, out_dtype=torch.float64))
    return engs, D.drive_lockstep(gens)


@pytest.mark.parametrize("G", [1, 2, 3])
def test_frame_routed_landmark_shards_match_unsharded(G, cuda_device):
    """Frame-routed landmark sharding: every rank screens only its home frames against the
    global coarse landmarks, frames travel to the shards their admissible tiles live on,
    gradient rows come back home.  The concatenated home outputs equal the unsharded
    evaluate (s, z to 1e-9; ds, dz to 1e-6 of the per-frame maximum)."""
    wl = synth.config4(T=260, L=1536, N=240)
    ref = engine.PathCVTC(wl.landmarks, wl.lam).evaluate(wl.frames, out_dtype=torch.float64)
    b = D.tile_bounds(1536, G)
    assert all(x % 48 == 0 for x in b[:-1])
    engs, outs = _routed(wl, G, b)
    s = torch.cat([o["s"] for o in outs]).cpu().numpy()
    z = torch.cat([o["z"] for o in outs]).cpu().numpy()
    np.testing.assert_allclose(s, ref["s"].cpu().numpy(), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(z, ref["z"].cpu().numpy(), rtol=1e-9, atol=1e-12)
    for key in ("ds", "dz"):
        got = torch.cat([o[key] for o in outs]).cpu().numpy()
        _rows_close(got, ref[key].cpu().numpy(), SHARD_REL)
    received = [o["received"] for o in outs]
    if G > 1:  # frames travel only where their hulls are: far fewer than G x T copies
        assert sum(received) < 1.6 * 260, received


def _two_phase(wl, G, bounds=None, routed=False, **kw):
    T = wl.frames.shape[0]
    if routed:  # routed phase 1: shards at landmark-tile bounds, the global coarse screen at home
        bounds = D.tile_bounds(wl.landmarks.shape[0], G)
        kw = dict(kw, route=True)
    engs = [engine.PathCVTC(wl.landmarks, wl.lam, shard=(g, G, bounds), two_phase=True, **kw) for g in range(G)]
    gens = []
    for g, e in enumerate(engs):
        off, cnt = D.shard_range(T, g, G)
        gens.append(e.two_phase_steps(wl.frames[off:off + cnt], off, T, out_dtype=torch.float64))
    return engs, D.drive_lockstep(gens)


@pytest.mark.parametrize("G,L,routed", [(1, 1536, False), (2, 1536, False), (3, 1536, False), (4, 768, False),
                                        (1, 1536, True), (2, 1536, True), (3, 1536, True), (4, 768, True)])
def test_two_phase_landmark_shards_match_unsharded(G, L, routed, cuda_device):
    """The two-phase plan (landmark-sharded screen, O(T) minima and windows; frame-sharded
    exact refits, weights and gradients against the replicated landmarks), with phase 1
    all-gathered (every frame's screening operand on every rank) or routed (each frame's
    operand only to the shards its coarse hull meets, windows back to the home rank): the
    concatenated home outputs equal the unsharded evaluate -- same windows, s and z to
    1e-9, ds and dz to SHARD_REL."""
    wl = synth.config4(T=260, L=L, N=240)
    ref = engine.PathCVTC(wl.landmarks, wl.lam).evaluate(wl.frames, out_dtype=torch.float64)
    engs, outs = _two_phase(wl, G, routed=routed)
    assert all(e.L < L for e in engs) or G == 1
    s = torch.cat([o["s"] for o in outs]).cpu().numpy()
    z = torch.cat([o["z"] for o in outs]).cpu().numpy()
    np.testing.assert_allclose(s, ref["s"].cpu().numpy(), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(z, ref["z"].cpu().numpy(), rtol=1e-9, atol=1e-12)
    lo = torch.cat([o["window_lo"] for o in outs]).cpu().numpy()
    cnt = torch.cat([o["window_cnt"] for o in outs]).cpu().numpy()
    rlo, rcnt = ref["window_lo"].cpu().numpy(), ref["window_cnt"].cpu().numpy()
    # the hull of the shards' windows covers the unsharded window (it can exceed it by the
    # unscanned margins of the banded screens at shard boundaries)
    assert (lo <= rlo).all() and (lo + cnt >= rlo + rcnt).all()
    assert cnt.sum() <= 1.05 * rcnt.sum()
    for key in ("ds", "dz"):
        got = torch.cat([o[key] for o in outs]).cpu().numpy()
        _rows_close(got, ref[key].cpu().numpy(), SHARD_REL)


def test_two_phase_through_nccl_one_rank(cuda_device):
    """evaluate_two_phase over a real NCCL process group (world size 1 on one GPU)."""
    wl = synth.config4(T=64, L=1536, N=240)
    init = not dist.is_initialized()
    if init:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=cuda_device)
    try:
        eng = engine.PathCVTC(wl.landmarks, wl.lam, shard=(0, 1), two_phase=True)
        out = eng.evaluate_two_phase(wl.frames, 0, 64, out_dtype=torch.float64)
        torch.cuda.synchronize()
    finally:
        if init:
            dist.destroy_process_group()
    ref = engine.PathCVTC(wl.landmarks, wl.lam).evaluate(wl.frames, out_dtype=torch.float64)
    np.testing.assert_allclose(out["s"].cpu().numpy(), ref["s"].cpu().numpy(), rtol=1e-9)
    _rows_close(out["ds"].cpu().numpy(), ref["ds"].cpu().numpy(), SHARD_REL)
