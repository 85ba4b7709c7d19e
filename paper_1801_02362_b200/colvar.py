"""Drop-in mirror of the SPEC colvar module: ReferenceSet,
CVResult and property_map (Eq. 2), plus the builder-defined path-CV z
(SURVEY.md A13).  The reduction runs in libmcb200 (mc_property_map)."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from ._lib import call, ptr, stream_ptr
from .errors import ConfigError, EmptyActiveSetError, InvalidStructureError


@dataclass
class ReferenceSet:
    """N centred reference structures, their properties q and lambda.

    q defaults to the reference index.  The device copy of the
    set (centred planes, norms, moments) is built once and cached.
    """

    structures: list
    properties: np.ndarray | None = None
    lam: float = 1.0
    _dev: dict = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if len(self.structures) < 1:
            raise EmptyActiveSetError("a reference set needs at least one structure")
        n = self.structures[0].n_atoms
        for i, s in enumerate(self.structures):
            if s.n_atoms != n:
                raise InvalidStructureError(f"reference {i} has {s.n_atoms} atoms, expected {n}")
        if self.properties is None:
            self.properties = np.arange(len(self.structures), dtype=float)
        self.properties = np.asarray(self.properties, dtype=float)
        if self.properties.shape != (len(self.structures),):
            raise ConfigError("one property per reference structure is required")
        if not (self.lam > 0):
            raise ConfigError("lambda must be positive")

    @property
    def n(self):
        return len(self.structures)

    def device(self, w, w_align):
        """Centred device planes of the set under the run's weights (cached)."""
        key = (w.tobytes(), w_align.tobytes())
        if self._dev is not None and self._dev.get("key") == key:
            return self._dev
        dev = torch.device("cuda", torch.cuda.current_device())
        coords = torch.from_numpy(np.stack([s.coords for s in self.structures])).to(dev)
        n = coords.shape[1]
        wd = torch.zeros(K.npad_for(n), dtype=torch.float64, device=dev)
        wad = torch.zeros_like(wd)
        wd[:n] = torch.from_numpy(w).to(dev)
        wad[:n] = torch.from_numpy(w_align).to(dev)
        c = K.center(coords, wad, wd, weighted=True, moments=True)
        self._dev = {"key": key, "c": c, "w": wd, "wa": wad,
                     "q": torch.from_numpy(self.properties).to(dev)}
        return self._dev


@dataclass
class CVResult:
    """CV value and its coordinate gradient; z/zgrad carry the path-CV z."""

    value: float
    grad: np.ndarray | None
    z: float | None = None
    zgrad: np.ndarray | None = None


def property_map(distances, ref: ReferenceSet) -> CVResult:
    """S = sum q_i e^{-lam D_i} / sum e^{-lam D_i} over the supplied active set,
    min-D stabilised, gradient by the quotient rule."""
    if len(distances) == 0:
        raise EmptyActiveSetError("property_map needs at least one distance")
    idx = np.array([i for i, _ in distances], dtype=np.int64)
    if np.any(idx < 0) or np.any(idx >= ref.n):
        raise ConfigError("reference index out of range")
    vals = np.array([float(d.value) for _, d in distances])
    if not np.all(np.isfinite(vals)):
        raise InvalidStructureError("non-finite distances")
    K.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    has_grad = all(d.grad is not None for _, d in distances)
    L = len(distances)
    D = torch.from_numpy(vals).to(dev)
    q = torch.from_numpy(ref.properties[idx]).to(dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    grads = ds = dz = None
    n = 0
    if has_grad:
        g = np.stack([np.asarray(d.grad, dtype=float) for _, d in distances])
        n = g.shape[1]
        grads = torch.from_numpy(g).to(dev)
        ds = torch.empty((n, 3), dtype=torch.float64, device=dev)
        dz = torch.empty((n, 3), dtype=torch.float64, device=dev)
    call("mc_property_map", L, n, ptr(D), ptr(grads), ptr(q), float(ref.lam), ptr(out), ptr(ds), ptr(dz),
         stream_ptr())
    o = out.cpu().numpy()
    return CVResult(float(o[0]), ds.cpu().numpy() if has_grad else None, float(o[1]),
                    dz.cpu().numpy() if has_grad else None)
