"""Seeded synthetic inputs for the five BASELINE.json configs.

The paper's cyclooctane / Trp-cage landmark sets and trajectories
 are not available, so every config is a seeded synthetic
stand-in with the shapes, sizes and value distributions BASELINE.json gives.
One generator feeds both the CUDA path and the CPU oracle, so parity never
depends on two RNG implementations.  Choices the config text leaves open are
fixed here and listed in DESIGN.md ("Synthetic inputs"):

* path parameter ``p`` is measured in landmark-index units, ``p in [0, L-1]``;
  the clean path point at ``p`` is the piecewise-linear interpolation between
  the endpoint conformations (landmark noise is *not* part of the path);
* random walks in ``p`` use a step of 0.5 landmark spacings and reflect at
  the ends;
* "random rigid motion" is an independent uniform rotation (normalised
  4-Gaussian quaternion) and a U(-1, 1)^3 nm translation per structure;
* config 1's "per-step coordinate noise" is fresh iid noise per frame (the
  literal reading; with it almost every frame exceeds eps);
* config 3's walkers accumulate their per-step noise (a random walk in
  coordinates) from a start on the path;
* lambda = 2.3 / mean aligned MSD of adjacent landmarks; eps = 0.1 x that
  mean (configs 1 and 3).

This module is data preparation, not part of the measured path: the adjacent
landmark MSD used for lambda/eps is a one-off numpy computation.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    frames: np.ndarray          # [T, N, 3] (config 3: [W, S, N, 3])
    landmarks: np.ndarray       # [L, N, 3]
    lam: float
    q: np.ndarray               # [L] property values (landmark index)
    eps: float | None = None    # close-structure threshold (configs 1, 3)
    meta: dict = field(default_factory=dict)


def random_rotations(rng, k):
    q = rng.standard_normal((k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q0, q1, q2, q3 = q.T
    return np.stack([
        np.stack([q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2)], -1),
        np.stack([2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1)], -1),
        np.stack([2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3], -1),
    ], -2)


def rigid_motion(rng, x, dtype=np.float64):
    """Apply an independent random rotation + U(-1,1)^3 translation per structure."""
    k = x.shape[0]
    rot = random_rotations(rng, k)
    trans = rng.uniform(-1.0, 1.0, size=(k, 1, 3))
    return (np.einsum("kab,kjb->kja", rot, x) + trans).astype(dtype)


def path_points(endpoints, p, n_landmarks):
    """Piecewise-linear path through the endpoints at landmark-unit parameter p."""
    n_seg = endpoints.shape[0] - 1
    u = np.clip(np.asarray(p, dtype=float) / (n_landmarks - 1), 0.0, 1.0) * n_seg
    seg = np.minimum(u.astype(np.int64), n_seg - 1)
    f = (u - seg)[:, None, None]
    return (1.0 - f) * endpoints[seg] + f * endpoints[seg + 1]


def make_landmarks(rng, endpoints, n_landmarks, noise=0.01, dtype=np.float64):
    base = path_points(endpoints, np.arange(n_landmarks), n_landmarks)
    base = base + rng.normal(0.0, noise, size=base.shape)
    return rigid_motion(rng, base, dtype)


def reflect_walk(rng, n_steps, n_landmarks, step=0.5, start=None):
    hi = float(n_landmarks - 1)
    p = np.empty(n_steps)
    cur = rng.uniform(0.0, hi) if start is None else start
    for t in range(n_steps):
        if t:
            cur = cur + rng.normal(0.0, step)
            while cur < 0.0 or cur > hi:
                cur = -cur if cur < 0.0 else 2.0 * hi - cur
        p[t] = cur
    return p


def _aligned_msd(x, a):
    """Minimal uniform-weight MSD of centred x vs a via Horn's 4x4 (numpy)."""
    n = x.shape[-2]
    xc = x - x.mean(axis=-2, keepdims=True)
    ac = a - a.mean(axis=-2, keepdims=True)
    s = np.einsum("...ja,...jb->...ab", ac, xc) / n
    gx = np.einsum("...ja,...ja->...", xc, xc) / n
    ga = np.einsum("...ja,...ja->...", ac, ac) / n
    sxx, sxy, sxz = s[..., 0, 0], s[..., 0, 1], s[..., 0, 2]
    syx, syy, syz = s[..., 1, 0], s[..., 1, 1], s[..., 1, 2]
    szx, szy, szz = s[..., 2, 0], s[..., 2, 1], s[..., 2, 2]
    h = np.stack([
        np.stack([sxx + syy + szz, syz - szy, szx - sxz, sxy - syx], -1),
        np.stack([syz - szy, sxx - syy - szz, sxy + syx, szx + sxz], -1),
        np.stack([szx - sxz, sxy + syx, -sxx + syy - szz, syz + szy], -1),
        np.stack([sxy - syx, szx + sxz, syz + szy, -sxx - syy + szz], -1),
    ], -2)
    lmax = np.linalg.eigvalsh(h)[..., -1]
    return gx + ga - 2.0 * lmax


def adjacent_msd(landmarks, chunk=256):
    lm = np.asarray(landmarks, dtype=float)
    vals = []
    for i in range(0, lm.shape[0] - 1, chunk):
        j = min(i + chunk, lm.shape[0] - 1)
        vals.append(_aligned_msd(lm[i + 1:j + 1], lm[i:j]))
    return float(np.mean(np.concatenate(vals)))


def _finish(name, frames, landmarks, eps_factor=None, meta=None):
    adj = adjacent_msd(landmarks)
    lam = 2.3 / adj
    q = np.arange(landmarks.shape[0], dtype=np.float64)
    eps = None if eps_factor is None else eps_factor * adj
    m = {"adjacent_msd": adj}
    m.update(meta or {})
    return Workload(name, frames, landmarks, lam, q, eps, m)


def config0(seed=0, T=1000, L=20, N=22):
    """Small path-CV: 2 endpoints, exact MSD, fp64."""
    rng = np.random.default_rng(seed)
    ends = rng.normal(0.0, 0.3, size=(2, N, 3))
    lms = make_landmarks(rng, ends, L)
    p = reflect_walk(rng, T, L)
    fr = path_points(ends, p, L) + rng.normal(0.0, 0.02, size=(T, N, 3))
    fr = rigid_motion(rng, fr)
    return _finish("config0", fr, lms, meta={"p": p})


def config1(seed=1, T=20000, L=500, N=304, noise=0.005, eps_factor=0.1):
    """Floating close structure: 3 endpoints, Brownian p, iid frame noise, fp64."""
    rng = np.random.default_rng(seed)
    ends = rng.normal(0.0, 0.3, size=(3, N, 3))
    lms = make_landmarks(rng, ends, L)
    p = reflect_walk(rng, T, L)
    fr = np.empty((T, N, 3))
    for t0 in range(0, T, 4096):
        t1 = min(T, t0 + 4096)
        blk = path_points(ends, p[t0:t1], L) + rng.normal(0.0, noise, size=(t1 - t0, N, 3))
        fr[t0:t1] = rigid_motion(rng, blk)
    return _finish("config1", fr, lms, eps_factor=eps_factor, meta={"p": p})


def _interp_frames(rng, ends, L, T, N, sigma_lo, sigma_hi, dtype, chunk=2048):
    fr = np.empty((T, N, 3), dtype=dtype)
    p = rng.uniform(0.0, L - 1, size=T)
    sig = np.exp(rng.uniform(math.log(sigma_lo), math.log(sigma_hi), size=T))
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        blk = path_points(ends, p[t0:t1], L)
        blk += rng.standard_normal(size=blk.shape) * sig[t0:t1, None, None]
        fr[t0:t1] = rigid_motion(rng, blk, dtype)
    return fr, p, sig


def config2(seed=2, T=65536, L=4096, N=1000, n_endpoints=16):
    """All-pairs MSD matrix: fp32 coords, sigma log-uniform in [1e-3, 0.5]."""
    rng = np.random.default_rng(seed)
    ends = rng.normal(0.0, 0.3, size=(n_endpoints, N, 3))
    lms = make_landmarks(rng, ends, L, dtype=np.float32)
    fr, p, sig = _interp_frames(rng, ends, L, T, N, 1e-3, 0.5, np.float32)
    return _finish("config2", fr, lms, meta={"p": p, "sigma": sig})


def config3(seed=3, W=256, N=2500, L=2048, steps=1000, step_noise=0.003, n_endpoints=2,
            eps_factor=0.1):
    """Multi-walker: per-walker accumulated random walk in coordinates, fp32.

    frames has shape [W, steps, N, 3]; landmarks "as in config 0" (2 endpoints).
    """
    rng = np.random.default_rng(seed)
    ends = rng.normal(0.0, 0.3, size=(n_endpoints, N, 3))
    lms = make_landmarks(rng, ends, L, dtype=np.float32)
    p0 = rng.uniform(0.0, L - 1, size=W)
    cur = path_points(ends, p0, L) + rng.normal(0.0, 0.02, size=(W, N, 3))
    fr = np.empty((W, steps, N, 3), dtype=np.float32)
    for s in range(steps):
        if s:
            cur = cur + rng.normal(0.0, step_noise, size=cur.shape)
        fr[:, s] = rigid_motion(rng, cur, np.float32)
    return _finish("config3", fr, lms, eps_factor=eps_factor, meta={"p0": p0})


def config4(seed=4, T=131072, L=8192, N=10000, n_endpoints=32):
    """Large sharded path: as config 2 with a 32-endpoint path."""
    rng = np.random.default_rng(seed)
    ends = rng.normal(0.0, 0.3, size=(n_endpoints, N, 3))
    lms = make_landmarks(rng, ends, L, dtype=np.float32)
    fr, p, sig = _interp_frames(rng, ends, L, T, N, 1e-3, 0.5, np.float32)
    return _finish("config4", fr, lms, meta={"p": p, "sigma": sig})


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def walkers_device(seed, W, steps, N, L, device, walker_offset=0, walker_count=None, step_noise=0.003,
                   n_endpoints=2, eps_factor=0.1):
    """Config 3 generated on the GPU: same distributions as ``config3`` (per-walker
    accumulated coordinate noise from a start on the path, fresh rigid motion per
    step).  Landmarks, lambda, eps and the walker starts come from numpy (seeded)
    so every rank agrees; walker w's trajectory is drawn from a generator seeded
    by (seed, w), so walker shards are slices of one global walker set."""
    import torch

    rng = np.random.default_rng(seed)
    ends = rng.normal(0.0, 0.3, size=(n_endpoints, N, 3))
    lms = make_landmarks(rng, ends, L, dtype=np.float32)
    p0 = rng.uniform(0.0, L - 1, size=W)
    wl = _finish(f"walkers{seed}", None, lms, eps_factor=eps_factor)
    walker_count = W - walker_offset if walker_count is None else walker_count
    starts = torch.from_numpy(path_points(ends, p0[walker_offset:walker_offset + walker_count], L)).to(device)
    frames = torch.empty((walker_count, steps, N, 3), dtype=torch.float32, device=device)
    for k in range(walker_count):
        g = torch.Generator(device=device).manual_seed(seed * 7_919 + walker_offset + k)
        start = starts[k] + torch.randn((N, 3), generator=g, device=device, dtype=torch.float64) * 0.02
        noise = torch.randn((steps, N, 3), generator=g, device=device, dtype=torch.float64) * step_noise
        noise[0] = 0.0
        cur = start[None] + torch.cumsum(noise, dim=0)
        q = torch.randn((steps, 4), generator=g, device=device, dtype=torch.float64)
        q = q / q.norm(dim=1, keepdim=True)
        q0, q1, q2, q3 = q.unbind(1)
        rot = torch.stack([
            torch.stack([q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2)], -1),
            torch.stack([2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1)], -1),
            torch.stack([2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3], -1),
        ], -2)
        trans = torch.rand((steps, 1, 3), generator=g, device=device, dtype=torch.float64) * 2 - 1
        frames[k] = (torch.einsum("kab,kjb->kja", rot, cur) + trans).float()
    wl.frames = frames
    wl.meta.update(generator="device (torch, per-walker seeded)", p0=p0)
    return wl


def interp_config_device(seed, T, L, N, n_endpoints, device, frame_offset=0, frame_count=None,
                         sigma_lo=1e-3, sigma_hi=0.5, chunk=4096):
    """Configs 2/4 generated on the GPU (torch RNG): same distributions as
    config2/config4 above, for full-size benchmark runs where host generation
    of 10^9..10^10 coordinates would dominate.  Landmarks and endpoints come
    from numpy (seeded) so lambda is identical on every rank; frames
    [frame_offset, frame_offset + frame_count) are drawn from a per-chunk
    seeded torch generator, so shards of a multi-GPU run are disjoint slices
    of one global frame set."""
    import torch

    rng = np.random.default_rng(seed)
    ends = rng.normal(0.0, 0.3, size=(n_endpoints, N, 3))
    lms = make_landmarks(rng, ends, L, dtype=np.float32)
    wl = _finish(f"device{seed}", None, lms)
    frame_count = T - frame_offset if frame_count is None else frame_count
    ends_t = torch.from_numpy(ends).to(device=device, dtype=torch.float32)
    frames = torch.empty((frame_count, N, 3), dtype=torch.float32, device=device)
    sigma = torch.empty((frame_count,), dtype=torch.float64, device=device)  # per-frame noise level
    n_seg = n_endpoints - 1
    for c0 in range(frame_offset - frame_offset % chunk, frame_offset + frame_count, chunk):
        g = torch.Generator(device=device).manual_seed(seed * 1_000_003 + c0 // chunk)
        cn = min(chunk, T - c0)
        p = torch.rand(cn, generator=g, device=device, dtype=torch.float64) * (L - 1)
        sig = torch.exp(torch.empty(cn, device=device, dtype=torch.float64).uniform_(
            math.log(sigma_lo), math.log(sigma_hi), generator=g))
        u = (p / (L - 1)).clamp(0, 1) * n_seg
        seg = u.long().clamp(max=n_seg - 1)
        f = (u - seg).float()[:, None, None]
        base = (1 - f) * ends_t[seg] + f * ends_t[seg + 1]
        base += torch.randn(base.shape, generator=g, device=device) * sig.float()[:, None, None]
        q = torch.randn((cn, 4), generator=g, device=device, dtype=torch.float64)
        q = q / q.norm(dim=1, keepdim=True)
        q0, q1, q2, q3 = q.unbind(1)
        rot = torch.stack([
            torch.stack([q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2)], -1),
            torch.stack([2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1)], -1),
            torch.stack([2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3], -1),
        ], -2).float()
        trans = (torch.rand((cn, 1, 3), generator=g, device=device) * 2 - 1)
        blk = torch.einsum("kab,kjb->kja", rot, base) + trans
        a = max(c0, frame_offset)
        b = min(c0 + cn, frame_offset + frame_count)
        if b > a:
            frames[a - frame_offset: b - frame_offset] = blk[a - c0: b - c0]
            sigma[a - frame_offset: b - frame_offset] = sig[a - c0: b - c0]
    wl.frames = frames
    wl.sigma = sigma
    wl.meta["generator"] = "device (torch, per-chunk seeded)"
    return wl
