"""World-size-2 gloo tests of the multi-GPU host logic (CPU, no GPU needed).

The per-rank compute is the CPU oracle on the rank's shard (standing in for
the device kernels, which cannot run here); what is tested is the sharding,
the exchange and the merge that the GPU ranks run with NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1801_02362_b200 import dist as D
from paper_1801_02362_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_shard_range_covers_disjointly():
    for total in (0, 1, 7, 131072, 131073):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                off, cnt = D.shard_range(total, r, world)
                seen.extend(range(off, off + cnt))
            assert seen == list(range(total))


def _landmark_sharded(rank, world):
    wl = synth.config0(seed=21, T=6, L=12, N=9)
    off, cnt = D.shard_range(wl.landmarks.shape[0], rank, world)
    loc = O.path_cv_exact(wl.frames, wl.landmarks[off:off + cnt], wl.lam, q=wl.q[off:off + cnt])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    s, z, ds, dz = D.merge_landmark_shards(t(loc["s"]), t(loc["z"]), wl.lam, t(loc["ds"]), t(loc["dz"]))
    return s.numpy(), z.numpy(), ds.numpy(), dz.numpy()


def test_landmark_sharded_lse_merge_matches_full():
    out = _spawn(_landmark_sharded)
    wl = synth.config0(seed=21, T=6, L=12, N=9)
    ref = O.path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    for rank in (0, 1):
        s, z, ds, dz = out[rank]
        np.testing.assert_allclose(s, ref["s"], rtol=1e-12)
        np.testing.assert_allclose(z, ref["z"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(ds, ref["ds"], atol=1e-10 * np.abs(ref["ds"]).max())
        np.testing.assert_allclose(dz, ref["dz"], atol=1e-10 * np.abs(ref["dz"]).max())
    # both ranks hold bitwise-identical merged values (fixed-order merge)
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def _frame_sharded(rank, world):
    wl = synth.config0(seed=22, T=9, L=7, N=8)
    off, cnt = D.shard_range(wl.frames.shape[0], rank, world)
    loc = O.batch_path_cv_exact(wl.frames[off:off + cnt], wl.landmarks, wl.lam)
    s = D.gather_frames(torch.from_numpy(loc["s"]), wl.frames.shape[0])
    ds = D.gather_frames(torch.from_numpy(loc["ds"]), wl.frames.shape[0])
    return s.numpy(), ds.numpy()


def test_frame_sharded_gather_matches_full():
    out = _spawn(_frame_sharded)
    wl = synth.config0(seed=22, T=9, L=7, N=8)
    ref = O.batch_path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    for rank in (0, 1):
        np.testing.assert_array_equal(out[rank][0], ref["s"])
        np.testing.assert_array_equal(out[rank][1], ref["ds"])


def test_merge_partials_single_shard_identity():
    s = torch.tensor([[1.5, 2.0]], dtype=torch.float64)
    z = torch.tensor([[0.3, 0.1]], dtype=torch.float64)
    ms, mz, w = D.merge_partials(s, z, 7.0)
    assert torch.equal(ms, s[0]) and torch.allclose(mz, z[0]) and torch.all(w == 1)
