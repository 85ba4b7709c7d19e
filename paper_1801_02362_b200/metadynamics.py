"""Metadynamics bias and bias force on the device (SPEC [MODULE] metadynamics,
PAPER Eq. 1).

``HillStore`` mirrors the spec's type: hills (centres s^{t'}, widths sigma,
height w, deposit step t') deposited every ``stride`` steps, with an optional
uniform grid per CV (d <= 2; cubic Hermite data: values, first derivatives and
the cross derivative) fed by 6-sigma-truncated depositions.  Evaluation is
batched over frames and consumes the path CVs and their atom gradients where
they already live: ``bias_and_force(cv [T, d], [ds, dz]) -> V [T], F [T, N, 3]``
with the physical sign F = -dV/dx (SPEC design decision; Eq. 1 prints +).
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import FLAG_OUT_OF_GRID, call, ptr, stream_ptr
from .errors import ConfigError, OutOfGridError

F64 = torch.float64


class HillStore:
    def __init__(self, d, stride, height, sigma, grid=None, cutoff=6.0, device=None):
        """d CVs (1..3); stride tau_G >= 1; constant height w >= 0 (Eq. 1, no
        well-tempering); sigma [d] > 0; grid = (lo [d], hi [d], bins [d]) or None
        (direct summation; grids support d <= 2)."""
        if not 1 <= int(d) <= 3:
            raise ConfigError("1 to 3 collective variables")
        if int(stride) < 1 or not (float(height) >= 0.0):
            raise ConfigError("stride >= 1 and height >= 0")
        self.d, self.stride, self.height, self.cutoff = int(d), int(stride), float(height), float(cutoff)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.sigma = torch.as_tensor(sigma, dtype=F64, device=self.device).reshape(self.d)
        if not bool((self.sigma > 0).all()):
            raise ConfigError("hill widths must be > 0")
        self.centers = torch.empty((0, self.d), dtype=F64, device=self.device)
        self.sigmas = torch.empty((0, self.d), dtype=F64, device=self.device)
        self.heights = torch.empty((0,), dtype=F64, device=self.device)
        self.steps = []
        self.grid = None
        if grid is not None:
            lo, hi, bins = grid
            if self.d > 2:
                raise ConfigError("bias grids support 1 or 2 CVs")
            import numpy as np

            self._lo = np.ascontiguousarray(np.asarray(lo, dtype=np.float64).reshape(self.d))
            self._hi = np.ascontiguousarray(np.asarray(hi, dtype=np.float64).reshape(self.d))
            self._bins = np.ascontiguousarray(np.asarray(bins, dtype=np.int32).reshape(self.d))
            if (self._hi <= self._lo).any() or (self._bins < 1).any():
                raise ConfigError("grid needs lo < hi and bins >= 1 per CV")
            shape = tuple(int(b) + 1 for b in self._bins)
            self.grid = {"val": torch.zeros(shape, dtype=F64, device=self.device),
                         "d": torch.zeros((self.d,) + shape, dtype=F64, device=self.device),
                         "dxy": torch.zeros(shape, dtype=F64, device=self.device) if self.d == 2 else None}
        self._flag = torch.zeros((1,), dtype=torch.uint8, device=self.device)

    def _geom(self):
        import ctypes

        return (self._lo.ctypes.data_as(ctypes.c_void_p), self._hi.ctypes.data_as(ctypes.c_void_p),
                self._bins.ctypes.data_as(ctypes.c_void_p))

    def deposit(self, cv_values, step):
        """Append a hill at cv_values [d] (device or host); step must be a multiple of
        the stride (SPEC pre).  With a grid, the hill is added to every node within
        6 sigma; a centre off the grid raises OutOfGridError."""
        if int(step) % self.stride:
            raise ConfigError(f"deposit at step {step}: not a multiple of the stride {self.stride}")
        if self.steps and int(step) < self.steps[-1]:
            raise ConfigError("hills are deposited in nondecreasing step order")
        c = torch.as_tensor(cv_values, dtype=F64).to(self.device).reshape(1, self.d)
        if self.grid is not None:
            # a rejected deposit must leave the grid untouched (grid and direct V agree for
            # every deposition history): check the centre before the kernel adds anything
            ch = c.cpu().numpy().reshape(self.d)
            if not ((ch >= self._lo) & (ch <= self._hi)).all():
                raise OutOfGridError("hill centre outside the bias grid")
            g = self.grid
            lo, hi, bins = self._geom()
            call("mc_mtd_grid_deposit", ptr(g["val"]), ptr(g["d"]), ptr(g["dxy"]), self.d, lo, hi, bins, ptr(c),
                 ptr(self.sigma), self.height, self.cutoff, ptr(self._flag), stream_ptr())
            if int(self._flag.item()) & FLAG_OUT_OF_GRID:
                raise OutOfGridError("hill centre outside the bias grid")
        self.centers = torch.cat([self.centers, c])
        self.sigmas = torch.cat([self.sigmas, self.sigma.reshape(1, self.d)])
        self.heights = torch.cat([self.heights, torch.full((1,), self.height, dtype=F64, device=self.device)])
        self.steps.append(int(step))
        return self

    def bias(self, cv, use_grid=None):
        """V [T] and dV/dS [T, d] at the frames' CV values cv [T, d] (device)."""
        cv = torch.as_tensor(cv, dtype=F64).to(self.device).reshape(-1, self.d).contiguous()
        T = cv.shape[0]
        V = torch.empty((T,), dtype=F64, device=self.device)
        dV = torch.empty((T, self.d), dtype=F64, device=self.device)
        grid = self.grid is not None if use_grid is None else use_grid
        if grid:
            g = self.grid
            flags = torch.empty((T,), dtype=torch.uint8, device=self.device)
            lo, hi, bins = self._geom()
            call("mc_mtd_grid_eval", ptr(g["val"]), ptr(g["d"]), ptr(g["dxy"]), self.d, lo, hi, bins, ptr(cv), T,
                 ptr(V), ptr(dV), ptr(flags), stream_ptr())
            if T and int(flags.max().item()) & FLAG_OUT_OF_GRID:
                raise OutOfGridError("collective variable outside the bias grid")
        else:
            call("mc_mtd_bias_direct", ptr(cv), T, self.d, ptr(self.centers), ptr(self.sigmas), ptr(self.heights),
                 self.centers.shape[0], ptr(V), ptr(dV), stream_ptr())
        return V, dV

    def bias_and_force(self, cv, grads, use_grid=None):
        """(V [T], F [T, N, 3]) with F = -sum_i dV/dS_i dS_i/dx; grads: d tensors [T, N, 3]
        (the CV atom gradients, e.g. path_cv's ds and dz), F in their dtype."""
        if len(grads) != self.d:
            raise ConfigError("one gradient tensor per collective variable")
        V, dV = self.bias(cv, use_grid)
        g = [x.contiguous() for x in grads]
        T, n = g[0].shape[0], g[0].shape[1]
        if any(x.shape != g[0].shape or x.dtype != g[0].dtype for x in g):
            raise ConfigError("CV gradients must share shape and dtype")
        F = torch.empty_like(g[0])
        dt = _lib.MC_F64 if g[0].dtype == torch.float64 else _lib.MC_F32
        call("mc_mtd_force", ptr(dV), T, self.d, ptr(g[0]), ptr(g[1] if self.d > 1 else None),
             ptr(g[2] if self.d > 2 else None), dt, n, ptr(F), stream_ptr())
        return V, F

    def write_hills(self, path):
        """HILLS file (SPEC external interface): one line per hill -- step, s_1..s_d,
        sigma_1..sigma_d, height -- space-separated, 17 significant digits."""
        c, s, h = self.centers.cpu().tolist(), self.sigmas.cpu().tolist(), self.heights.cpu().tolist()
        with open(path, "w") as f:
            for k, step in enumerate(self.steps):
                vals = [f"{v:.17g}" for v in (*c[k], *s[k], h[k])]
                f.write(" ".join([str(step)] + vals) + "\n")
