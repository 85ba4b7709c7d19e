"""Toy MD driver on the device (SPEC [MODULE] toysim).

Mirror of the spec's types and operation:

* ``ToySystem`` — n_beads, bond_k, bond_r0, angle_k, temperature, friction, dt,
  rng_seed plus the two constants the spec leaves open: bead
  mass (amu) and the angle's equilibrium theta0 (rad).
* ``RunReport`` — steps, mode, expensive / cheap / reassign counts, measured K,
  the CV series (s per step), the bias series, wall time;
  plus z, D(x, y) and the per-step reassignment log.
* ``run(system, ref, mode, nl_config, mtd_config, n_steps)`` and
  the batched ``ToySim`` (W independent walkers, one CTA each, the whole
  trajectory in one launch of ``mc_toysim_run``; state kept on the device so a
  run can continue in chunks).
* ``make_references`` — the seeded unbiased pre-run snapshotted at fixed
  intervals, then centred, q_i = i.

Neighbour list (``nl_config``: a ``neighbourlist.NeighbourList`` or an object with
``size`` M, ``stride`` L and ``enabled``): each walker keeps its own
list on the device, updated on the first step and whenever step − last_update ≥ L from
that step's distances to all N references (exact in the original mode, the Eq. 5
approximations in the close mode), the M smallest with ties by the lower index; between
updates only the M members are evaluated and s, z and the bias force sum over them.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from ._lib import FLAG_NO_CONVERGE, FLAG_NON_FINITE, FLAG_SIG_OVERFLOW, call, ptr, stream_ptr
from .errors import ConfigError, InvalidStructureError, MetadynError

KB = 0.0083144626  # kJ/mol/K
F64 = torch.float64
MODES = {"free": 0, "original": 1, "close": 2}


@dataclass
class ToySystem:
    n_beads: int = 8
    bond_k: float = 2000.0  # kJ/mol/nm^2
    bond_r0: float = 0.15  # nm
    angle_k: float = 100.0  # kJ/mol/rad^2
    temperature: float = 300.0  # K
    friction: float = 10.0  # 1/ps
    dt: float = 1e-3  # ps
    rng_seed: int = 0
    mass: float = 12.0  # amu (not in the SPEC type; overdamped mobility dt / (m gamma))
    theta0: float = 1.9106332362490186  # rad (tetrahedral; not in the SPEC type)

    def __post_init__(self):
        if int(self.n_beads) < 3 or int(self.n_beads) > 64:
            raise ConfigError("3 <= n_beads <= 64")
        if not (self.dt > 0 and self.temperature >= 0 and self.friction > 0 and self.mass > 0):
            raise ConfigError("dt > 0, temperature >= 0, friction > 0, mass > 0 (SPEC.md:316)")

    @property
    def mobility(self):
        return self.dt / (self.mass * self.friction)

    @property
    def noise(self):
        return math.sqrt(2.0 * KB * self.temperature * self.mobility)

    def initial_chain(self):
        """Planar zig-zag at bond length r0 and angle theta0 (a zero-force configuration)."""
        n = int(self.n_beads)
        half = 0.5 * self.theta0
        dx, dy = self.bond_r0 * math.sin(half), self.bond_r0 * math.cos(half)
        x = np.zeros((n, 3))
        for k in range(1, n):
            x[k] = x[k - 1] + np.array([dx, dy if k % 2 else -dy, 0.0])
        return x


@dataclass
class MtdConfig:
    tau_g: int = 50
    sigma: float = 0.5
    height: float = 0.5  # kJ/mol
    max_hills: int = 0  # 0: n_steps // tau_g + 1


@dataclass
class RunReport:
    steps: int
    mode: str
    expensive_count: int
    cheap_count: int
    reassign_count: int
    measured_K: float
    cv_series: np.ndarray
    bias_series: np.ndarray
    z_series: np.ndarray
    dxy_series: np.ndarray
    refresh_log: np.ndarray
    wall_time: float
    final_coords: np.ndarray = field(repr=False, default=None)
    trajectory: np.ndarray = field(repr=False, default=None)  # [frames, n, 3] every traj_stride steps
    traj_stride: int = 0

    # SPEC toysim "External Interfaces"
    def write_cv_csv(self, path):
        """CV series: CSV "step,cv_value,bias", one row per step."""
        with open(path, "w") as f:
            f.write("step,cv_value,bias\n")
            for k, (c, b) in enumerate(zip(self.cv_series, self.bias_series)):
                f.write(f"{k},{float(c)!r},{float(b)!r}\n")

    def write_trajectory(self, path):
        """Trajectory: plain-text frames -- the step, then n_beads lines "x y z"."""
        if self.trajectory is None:
            raise ConfigError("no trajectory recorded (run with traj_stride > 0)")
        with open(path, "w") as f:
            for k, x in enumerate(self.trajectory):
                f.write(f"{k * self.traj_stride}\n")
                for r in x:
                    f.write(f"{float(r[0])!r} {float(r[1])!r} {float(r[2])!r}\n")

    def counter_report(self):
        """The counters the SPEC perf identities are checked against."""
        return {"steps": self.steps, "mode": self.mode, "expensive_count": self.expensive_count,
                "cheap_count": self.cheap_count, "reassign_count": self.reassign_count,
                "measured_K": self.measured_K, "expensive_per_step": self.expensive_count / max(1, self.steps)}


class ToySim:
    """W walkers of one ToySystem against one reference set, state on the device."""

    def __init__(self, system: ToySystem, refs, mode="close", lam=100.0, eps=0.01, mtd: MtdConfig | None = None,
                 walkers=1, x0=None, q=None, max_hills=1024, device=None, nl_config=None):
        K.require_cuda()
        if mode not in MODES:
            raise ConfigError(f"mode {mode!r}")
        self.sys, self.mode, self.W = system, mode, int(walkers)
        self.lam, self.eps = float(lam), float(eps)
        self.mtd = mtd or MtdConfig()
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        n = int(system.n_beads)
        self.n = n
        if mode != "free":
            r = np.asarray(refs, dtype=np.float64)
            if r.ndim != 3 or r.shape[1:] != (n, 3):
                raise InvalidStructureError("references must be [L, n_beads, 3] (SPEC.md:326 atom-count match)")
            if not 1 <= r.shape[0] <= 128:
                raise ConfigError("1 <= L <= 128 references")
            w = np.full(n, 1.0 / n)
            r = r - np.einsum("j,ljk->lk", w, r)[:, None, :]  # centred
            self.L = r.shape[0]
            self.refs = torch.from_numpy(np.ascontiguousarray(r)).to(self.dev)
            self.refg = torch.from_numpy(np.einsum("j,ljk,ljk->l", w, r, r)).to(self.dev)
            m = np.einsum("j,ljb,ljg->lbg", w, r, r)
            self.refmom = torch.from_numpy(np.ascontiguousarray(
                np.stack([m[:, 0, 0], m[:, 0, 1], m[:, 0, 2], m[:, 1, 1], m[:, 1, 2], m[:, 2, 2]], axis=1))).to(self.dev)
            qq = np.arange(self.L, dtype=np.float64) if q is None else np.asarray(q, dtype=np.float64)
            if qq.shape != (self.L,):
                raise ConfigError("q must have one value per reference")
            self.q = torch.from_numpy(qq).to(self.dev)
        else:
            self.L = 1
            self.refs = self.refg = self.refmom = self.q = None
        self.w = torch.full((n,), 1.0 / n, dtype=F64, device=self.dev)
        x = system.initial_chain() if x0 is None else np.asarray(x0, dtype=np.float64)
        x = np.repeat(x[None], self.W, axis=0) if x.ndim == 2 else x
        if x.shape != (self.W, n, 3):
            raise InvalidStructureError("x0 must be [n, 3] or [walkers, n, 3]")
        self.x = torch.from_numpy(np.ascontiguousarray(x)).to(self.dev)
        self.y = torch.zeros_like(self.x)
        self.rays = torch.zeros((self.W, self.L, 9), dtype=F64, device=self.dev)
        self.hasy = torch.zeros((self.W,), dtype=torch.int32, device=self.dev)
        self.max_hills = int(max_hills)
        self.hills = torch.zeros((self.W, max(1, self.max_hills)), dtype=F64, device=self.dev)
        self.nhills = torch.zeros((self.W,), dtype=torch.int32, device=self.dev)
        self.counters = torch.zeros((self.W, 3), dtype=torch.int64, device=self.dev)
        self.flags = torch.zeros((self.W,), dtype=torch.uint8, device=self.dev)
        self.step = 0
        # neighbour list (SPEC neighbourlist): M, stride; per-walker members + last update
        self.nl_m, self.nl_stride = 0, 1
        if nl_config is not None and getattr(nl_config, "enabled", True):
            if mode == "free":
                raise ConfigError("a neighbour list needs the path CV (mode original or close)")
            m, st = int(nl_config.size), int(getattr(nl_config, "stride", 1))
            if not 1 <= m <= self.L:
                raise ConfigError("neighbour list size must satisfy 1 <= M <= N")
            if st < 1:
                raise ConfigError("neighbour list stride must be >= 1")
            self.nl_m, self.nl_stride = m, st
        self.act = torch.zeros((self.W, self.L), dtype=torch.uint8, device=self.dev)
        self.nl_last = torch.full((self.W,), -1, dtype=torch.int64, device=self.dev)

    def run(self, n_steps, traj_stride=0):
        """Advance every walker n_steps (one launch).  Returns a dict of device tensors:
        cv [W, steps, 4] = (s, z, V_bias, D(x, y)), refresh [W, steps] and traj."""
        n_steps = int(n_steps)
        cv = torch.empty((self.W, max(1, n_steps), 4), dtype=F64, device=self.dev)
        rlog = torch.empty((self.W, max(1, n_steps)), dtype=torch.uint8, device=self.dev)
        traj = None
        if traj_stride:
            if self.step % traj_stride:
                raise ConfigError("continue a trajectory run at a multiple of traj_stride")
            traj = torch.empty((self.W, (n_steps + traj_stride - 1) // traj_stride, self.n, 3), dtype=F64,
                               device=self.dev)
        s = self.sys
        call("mc_toysim_run", self.W, self.n, self.L, n_steps, self.step, MODES[self.mode], int(self.mtd.tau_g),
             self.max_hills, int(traj_stride), float(s.bond_k), float(s.bond_r0), float(s.angle_k), float(s.theta0),
             float(s.mobility), float(s.noise), self.lam, self.eps, float(self.mtd.height), float(self.mtd.sigma),
             int(s.rng_seed) & 0xFFFFFFFFFFFFFFFF, ptr(self.refs), ptr(self.refg), ptr(self.refmom), ptr(self.q),
             ptr(self.w), ptr(self.w), ptr(self.x), ptr(self.y), ptr(self.rays), ptr(self.hasy), ptr(self.hills),
             ptr(self.nhills), ptr(self.counters), ptr(cv), ptr(rlog), ptr(traj), ptr(self.flags), self.nl_m,
             self.nl_stride, ptr(self.act), ptr(self.nl_last), stream_ptr())
        self.step += n_steps
        return {"cv": cv[:, :n_steps], "refresh": rlog[:, :n_steps], "traj": traj}

    def check(self):
        """Raise on the device status bits of any walker (one host read)."""
        bits = 0
        for v in self.flags.cpu().tolist():
            bits |= v
        if bits & FLAG_NON_FINITE:
            raise InvalidStructureError("toysim: non-finite coordinates or CV (time step too large?)")
        if bits & FLAG_NO_CONVERGE:
            raise MetadynError("toysim: Jacobi diagonalisation did not converge")
        if bits & FLAG_SIG_OVERFLOW:
            raise ConfigError("toysim: hill capacity exceeded (raise max_hills)")
        return bits


def make_references(system: ToySystem, n_refs=16, stride=200, warmup=0, walker=0):
    """Unbiased pre-run snapshotted every ``stride`` steps (after ``warmup`` steps,
    rounded up to a multiple of the stride), centred."""
    sim = ToySim(system, None, mode="free", walkers=walker + 1)
    if warmup:
        sim.run(-(-int(warmup) // stride) * stride)
    out = sim.run(n_refs * stride, traj_stride=stride)
    sim.check()
    refs = out["traj"][walker].cpu().numpy()
    return refs - refs.mean(axis=1, keepdims=True)


def run(system: ToySystem, ref, mode="close", nl_config=None, mtd_config: MtdConfig | None = None, n_steps=5000,
        lam=100.0, eps=0.01, traj_stride=0):
    """SPEC toysim.run: one walker, returns a RunReport."""
    refs = ref.coords if hasattr(ref, "coords") else ref
    mtd = mtd_config or MtdConfig()
    cap = mtd.max_hills or (n_steps // max(1, mtd.tau_g) + 1)
    sim = ToySim(system, refs, mode=mode, lam=lam, eps=eps, mtd=mtd, walkers=1, max_hills=cap, nl_config=nl_config)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = sim.run(n_steps, traj_stride=traj_stride)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    sim.check()
    cv = out["cv"][0].cpu().numpy()
    c = sim.counters[0].cpu().tolist()
    reas = int(c[2])
    return RunReport(steps=n_steps, mode=mode, expensive_count=int(c[0]), cheap_count=int(c[1]), reassign_count=reas,
                     measured_K=(n_steps / reas) if reas else float("inf"), cv_series=cv[:, 0], bias_series=cv[:, 2],
                     z_series=cv[:, 1], dxy_series=cv[:, 3], refresh_log=out["refresh"][0].cpu().numpy(),
                     wall_time=wall, final_coords=sim.x[0].cpu().numpy(),
                     trajectory=None if out["traj"] is None else out["traj"][0].cpu().numpy(),
                     traj_stride=int(traj_stride))
