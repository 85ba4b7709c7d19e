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


# ---------------------------------------------------------------- landmark-sharded exchanges
#
# The same collective sequence as PathCVTC.sharded_steps (min -> gather -> exchange),
# with the oracle's exact distances and gradients standing in for the device
# kernels: per-shard windows against the global minimum, local (s_g, z_g), the
# (alpha, beta) coefficient rescaling and the owner all-to-all of the gradient rows.

_CUT = 6.0  # small, so that the toy path's windows split between the shards


def _toy_problem():
    wl = synth.config0(seed=5, T=40, L=16, N=7)  # frames near landmarks 7..14: both shards
    n = wl.frames.shape[1]
    w = O.normalise_weights(None, n)
    lc = np.stack([O.center(a, w) for a in wl.landmarks])
    D_ = np.zeros((wl.frames.shape[0], wl.landmarks.shape[0]))
    G_ = np.zeros(D_.shape + (n, 3))
    for t, x in enumerate(wl.frames):
        xc = O.center(x, w)
        for i in range(lc.shape[0]):
            D_[t, i], G_[t, i], _ = O.exact_distance(xc, lc[i], w, w, with_rot_term=False)
    return wl, D_, G_


def _toy_steps(rank, world, wl, D_, G_, cut=_CUT):
    """Generator mirroring PathCVTC.sharded_steps on precomputed D / dD."""
    T, L = D_.shape
    off, cnt = D.shard_range(L, rank, world)
    Dl = torch.from_numpy(D_[:, off:off + cnt].copy())
    Gl = torch.from_numpy(G_[:, off:off + cnt].copy())
    q = torch.arange(off, off + cnt, dtype=torch.float64)
    lam = wl.lam
    dref = yield ("min", Dl.min(1).values)
    win = lam * (Dl - dref[:, None]) <= cut
    sl = torch.zeros(T, dtype=torch.float64)
    zl = torch.full((T,), float("inf"), dtype=torch.float64)
    cs = torch.zeros((T, cnt), dtype=torch.float64)
    cz = torch.zeros((T, cnt), dtype=torch.float64)
    for t in range(T):
        if not win[t].any():
            continue
        d = Dl[t][win[t]]
        e = torch.exp(-lam * (d - d.min()))
        p = e / e.sum()
        sl[t] = (p * q[win[t]]).sum()
        zl[t] = d.min() - torch.log(e.sum()) / lam
        cs[t, win[t]] = -lam * p * (q[win[t]] - sl[t])
        cz[t, win[t]] = p
    parts = yield ("gather", torch.cat([sl, zl]))
    s_parts, z_parts = parts[:, :T], parts[:, T:]
    s, z, alpha, beta = D.shard_coefficients(s_parts, z_parts, lam, rank)
    cs2 = alpha[:, None] * (cs + beta[:, None] * cz)
    cz2 = alpha[:, None] * cz
    ds = torch.einsum("ti,tika->tka", cs2, Gl)
    dz = torch.einsum("ti,tika->tka", cz2, Gl)
    owner = yield ("exchange", ds, dz, z_parts)
    return {"s": s, "z": z, "ds": ds, "dz": dz, "owner": owner, "z_parts": z_parts}


def _sharded_exchange(rank, world):
    wl, D_, G_ = _toy_problem()
    out = D.drive(_toy_steps(rank, world, wl, D_, G_), D.DistComm())
    return {k: v.numpy() for k, v in out.items()}


def test_landmark_sharded_exchange_matches_full():
    out = _spawn(_sharded_exchange)
    wl, D_, G_ = _toy_problem()
    # one shard with the same truncation is the reference; untruncated it is the oracle
    ref = {k: v.numpy() for k, v in D.drive_lockstep([_toy_steps(0, 1, wl, D_, G_)])[0].items()}
    full = D.drive_lockstep([_toy_steps(0, 1, wl, D_, G_, cut=1e9)])[0]
    orc = O.batch_path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    np.testing.assert_allclose(full["s"].numpy(), orc["s"], rtol=1e-12)
    np.testing.assert_allclose(full["ds"].numpy(), orc["ds"], atol=1e-10 * np.abs(orc["ds"]).max())
    owner = out[0]["owner"]
    assert np.array_equal(owner, out[1]["owner"])
    zp = out[0]["z_parts"]
    # the windows really are split: some frames are empty on one shard, some straddle
    assert (~np.isfinite(zp)).any() and np.isfinite(zp).all(0).any()
    for rank in (0, 1):
        o = out[rank]
        np.testing.assert_allclose(o["s"], ref["s"], rtol=1e-12)
        np.testing.assert_allclose(o["z"], ref["z"], rtol=1e-12, atol=1e-15)
        mine = owner == rank
        for key in ("ds", "dz"):
            np.testing.assert_allclose(o[key][mine], ref[key][mine], atol=1e-10 * np.abs(ref[key]).max())
    # the lock-step single-process driver (used by the one-GPU tests) gives the same bits
    loc = D.drive_lockstep([_toy_steps(r, 2, wl, D_, G_) for r in range(2)])
    for rank in (0, 1):
        for key in ("s", "z", "owner"):
            assert np.array_equal(loc[rank][key].numpy(), out[rank][key])
        mine = owner == rank
        for key in ("ds", "dz"):
            assert np.array_equal(loc[rank][key].numpy()[mine], out[rank][key][mine])


def test_merge_partials_empty_shard():
    s = torch.tensor([[1.5, 0.0], [2.5, 3.0]], dtype=torch.float64)
    z = torch.tensor([[0.3, float("inf")], [0.3, 0.1]], dtype=torch.float64)
    ms, mz, w = D.merge_partials(s, z, 7.0)
    assert w[0, 1] == 0 and w[1, 1] == 1 and ms[1] == 3.0 and mz[1] == 0.1
    np.testing.assert_allclose(w[:, 0].numpy(), [0.5, 0.5])
    assert D.gradient_owners(z).tolist() == [0, 1]


def test_balanced_bounds():
    b = D.balanced_bounds(torch.ones(10), 3)
    assert b == [0, 4, 7, 10]
    load = torch.zeros(64)
    load[10:14] = 1000.0  # one hot region
    b = D.balanced_bounds(load, 4)
    assert b[0] == 0 and b[-1] == 64 and all(x < y for x, y in zip(b, b[1:]))
    assert sum(1 for x in b[1:-1] if 10 <= x <= 14) >= 2  # the hot region is split
    assert D.balanced_bounds(torch.zeros(4), 4) == [0, 1, 2, 3, 4]


def _toy_alltoallv(rank, world):
    """Variable-size all-to-all of two fields (int64 ids, float rows)."""
    def steps(r):
        ids = [torch.arange(r * 10 + d, r * 10 + d + d + r, dtype=torch.int64) for d in range(world)]
        rows = [torch.full((int(i.numel()), 2, 3), float(r * 100 + d)) for d, i in enumerate(ids)]
        got = yield ("alltoallv", [ids, rows])
        return {"ids": torch.cat(got[0]), "rows": torch.cat(got[1])}
    out = D.drive(steps(rank), D.DistComm())
    return {k: v.numpy() for k, v in out.items()}


def test_alltoallv_dist_equals_lockstep():
    out = _spawn(_toy_alltoallv)

    def steps(r, world=2):
        ids = [torch.arange(r * 10 + d, r * 10 + d + d + r, dtype=torch.int64) for d in range(world)]
        rows = [torch.full((int(i.numel()), 2, 3), float(r * 100 + d)) for d, i in enumerate(ids)]
        got = yield ("alltoallv", [ids, rows])
        return {"ids": torch.cat(got[0]), "rows": torch.cat(got[1])}

    loc = D.drive_lockstep([steps(0), steps(1)])
    for r in (0, 1):
        assert np.array_equal(loc[r]["ids"].numpy(), out[r]["ids"])
        assert np.array_equal(loc[r]["rows"].numpy(), out[r]["rows"])
    # rank 1 receives rank 0's block for destination 1 ([1]) then its own ([11, 12])
    assert out[1]["ids"].tolist() == [1, 11, 12]


def test_tile_bounds():
    assert D.tile_bounds(1536, 1) == [0, 1536]
    b = D.tile_bounds(1536, 3)
    assert b == [0, 528, 1056, 1536] or all(x % 48 == 0 for x in b[:-1])
    b = D.tile_bounds(1000, 4)
    assert b[0] == 0 and b[-1] == 1000 and all(x % 48 == 0 for x in b[:-1])


def _two_phase(rank, world):
    """The two-phase landmark-sharded protocol (PathCVTC.two_phase_steps) with the oracle's
    exact distances standing in for the device screen: ragged all-gather of the frames'
    screening operand (DistComm.allgather_split), all-reduce MIN of the per-frame minimum,
    all-gather of every shard's windows, hull merge, phase-2 exact path CV of the home
    frames over the merged windows."""
    from paper_1801_02362_b200.kernels import Split

    wl = synth.config0(seed=23, T=7, L=16, N=9)
    T, L, n = wl.frames.shape[0], wl.landmarks.shape[0], wl.frames.shape[1]
    comm = D.DistComm()
    off, cnt = D.shard_range(T, rank, world)
    b = D.balanced_bounds(torch.ones(L), world)
    l0, l1 = b[rank], b[rank + 1]
    # the home frames' "split": coordinates as halves in plane-major [3, count, n] + scalars
    home = wl.frames[off:off + cnt]
    hi = torch.from_numpy(np.ascontiguousarray(home.transpose(2, 0, 1))).half()
    sc = torch.from_numpy(np.arange(off, off + cnt, dtype=np.float64))
    sp = Split(hi, None, sc[:, None].repeat(1, 3), sc, sc[:, None].repeat(1, 3), None,
               torch.zeros(cnt, dtype=torch.uint8), n, n, sc, "f16", 1, sc, sc)
    allsp, counts = comm.allgather_split(sp)
    assert counts == [D.shard_range(T, r, world)[1] for r in range(world)]
    got_hi = allsp.hi.float().numpy().transpose(1, 2, 0)
    assert allsp.count == T and np.array_equal(allsp.g.numpy(), np.arange(T, dtype=np.float64))
    assert np.array_equal(got_hi, wl.frames.astype(np.float16).astype(np.float32))
    # phase 1: every frame against this landmark shard
    fc = O.batch_center(wl.frames, np.full(n, 1.0 / n))
    lc = O.batch_center(wl.landmarks, np.full(n, 1.0 / n))
    Dsh = O.batch_fit(fc[:, None], lc[None, l0:l1], np.full(n, 1.0 / n))[0][..., 0]  # [T, l1 - l0]
    dmin = comm.min(torch.from_numpy(Dsh.min(axis=1)))
    thr = 12.0
    lo = np.zeros(T, dtype=np.int32)
    cn = np.zeros(T, dtype=np.int32)
    for t in range(T):
        ok = np.nonzero(wl.lam * (Dsh[t] - dmin[t].item()) <= thr)[0]
        if ok.size:
            lo[t], cn[t] = l0 + ok[0], ok[-1] - ok[0] + 1
    parts = comm.gather(torch.from_numpy(np.stack([lo, cn])))
    glo, gcn = parts[:, 0].long(), parts[:, 1].long()
    act = gcn > 0
    lo_t = torch.where(act, glo, torch.full_like(glo, 1 << 40)).amin(0).numpy()
    hi_t = torch.where(act, glo + gcn, torch.full_like(glo, -1)).amax(0).numpy()
    # phase 2: the home frames over their merged windows
    res = []
    for t in range(off, off + cnt):
        a, e = int(lo_t[t]), int(hi_t[t])
        r = O.path_cv_exact(wl.frames[t:t + 1], wl.landmarks[a:e], wl.lam, q=wl.q[a:e])
        res.append((a, e, r["s"][0], r["z"][0], r["ds"][0], r["dz"][0]))
    return lo_t, hi_t, res


def test_two_phase_landmark_sharding_protocol():
    out = _spawn(_two_phase)
    wl = synth.config0(seed=23, T=7, L=16, N=9)
    T, n = wl.frames.shape[0], wl.frames.shape[1]
    ref = O.path_cv_exact(wl.frames, wl.landmarks, wl.lam)
    fc = O.batch_center(wl.frames, np.full(n, 1.0 / n))
    lc = O.batch_center(wl.landmarks, np.full(n, 1.0 / n))
    Dfull = O.batch_fit(fc[:, None], lc[None], np.full(n, 1.0 / n))[0][..., 0]
    # the merged windows are the unsharded windows (hull of the same global threshold)
    for t in range(T):
        ok = np.nonzero(wl.lam * (Dfull[t] - Dfull[t].min()) <= 12.0)[0]
        for r in (0, 1):
            assert (out[r][0][t], out[r][1][t]) == (ok[0], ok[-1] + 1)
    t = 0
    for r in (0, 1):
        for a, e, s, z, ds, dz in out[r][2]:
            # landmarks outside the window weigh < e^-12 of the leading term
            assert abs(s - ref["s"][t]) <= 1e-4 * max(1.0, abs(ref["s"][t]))
            assert abs(z - ref["z"][t]) <= 1e-4 * abs(ref["z"][t]) + 1e-7
            assert np.abs(ds - ref["ds"][t]).max() <= 1e-3 * np.abs(ref["ds"][t]).max()
            t += 1
    assert t == T
