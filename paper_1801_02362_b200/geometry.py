"""Drop-in mirror of the reference geometry module
(/root/reference/pkg/src/metadyn_close/geometry.py) backed by libmcb200.

Same names, argument meaning and errors:
  Structure (geometry.py:25-80), center (:83), RotationFit (:87-103),
  jacobi_eigh (:106), kearsley_fit (:227), rotation_derivative_check (:266).
Argument validation and the immutable host data type stay on the host like
the reference; every arithmetic step (centroid, centring, Kearsley form,
eigen-solve, rotation, dR/dx) runs in the CUDA library.  ``kearsley_fit_batch``
is the batched form the hot path uses.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from ._lib import FLAG_DEGENERATE, FLAG_NO_CONVERGE
from .errors import ConfigError, DegenerateFitError, InvalidStructureError

CENTER_TOL = 1e-12      # geometry.py:21
DEGENERACY_TOL = 1e-9   # geometry.py:22


def _device():
    K.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _wdev(w, n, dev):
    out = torch.zeros(K.npad_for(n), dtype=torch.float64, device=dev)
    out[:n] = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float64)).to(dev)
    return out


class Structure:
    """Atom coordinates (nm) with displacement and alignment weights.

    Weights are normalised to sum to one on construction; arrays are copied
    and read-only (geometry.py:25-47).
    """

    __slots__ = ("coords", "disp_weights", "align_weights")

    def __init__(self, coords, disp_weights=None, align_weights=None):
        coords = np.array(coords, dtype=float)
        if coords.ndim != 2 or coords.shape[1] != 3:
            raise InvalidStructureError(f"coords must be (n, 3), got {coords.shape}")
        n = coords.shape[0]
        if n < 2:
            raise InvalidStructureError("a structure needs at least 2 atoms")
        if not np.all(np.isfinite(coords)):
            raise InvalidStructureError("coords contain non-finite values")
        self.coords = coords
        self.disp_weights = self._normalise(disp_weights, n, "displacement")
        self.align_weights = self._normalise(align_weights, n, "alignment")
        for arr in (self.coords, self.disp_weights, self.align_weights):
            arr.flags.writeable = False

    @staticmethod
    def _normalise(w, n, kind):
        if w is None:
            return np.full(n, 1.0 / n)
        w = np.array(w, dtype=float)
        if w.shape != (n,):
            raise InvalidStructureError(f"{kind} weights must have length {n}")
        if not np.all(np.isfinite(w)) or np.any(w < 0.0):
            raise InvalidStructureError(f"{kind} weights must be finite and non-negative")
        total = w.sum()
        if total <= 0.0:
            raise InvalidStructureError(f"{kind} weights sum to zero")
        return w / total

    @property
    def n_atoms(self):
        return self.coords.shape[0]

    def _centred_device(self):
        dev = _device()
        x = torch.from_numpy(np.array(self.coords))[None].to(dev)
        n = self.n_atoms
        return K.center(x, _wdev(self.align_weights, n, dev), _wdev(self.disp_weights, n, dev))

    def centroid(self):
        """Alignment-weighted centroid (geometry.py:67-69), computed on device."""
        return self._centred_device().centroid[0].cpu().numpy()

    def is_centered(self, tol=CENTER_TOL):
        return bool(np.all(np.abs(self.centroid()) <= tol))

    def center(self):
        """Copy shifted so the alignment-weighted centroid is zero (geometry.py:74-76)."""
        c = self._centred_device()
        return self.with_coords(c.planes[0, :, : self.n_atoms].T.cpu().numpy())

    def with_coords(self, coords):
        return Structure(coords, self.disp_weights, self.align_weights)


def center(s: Structure) -> Structure:
    return s.center()


@dataclass(frozen=True)
class RotationFit:
    """rot maps the reference onto the fitted structure; quat is scalar-first;
    eigvals ascending (eigvals[0] = minimal weighted MSD); rot_grad[k, alpha]
    = dR/dx_{k,alpha} or None (geometry.py:87-103)."""

    rot: np.ndarray
    quat: np.ndarray
    eigvals: np.ndarray
    rot_grad: np.ndarray | None = None


def jacobi_eigh(mat, tol=1e-14, max_sweeps=60):
    """Cyclic-Jacobi eigen-decomposition (geometry.py:106-153) of a symmetric matrix on
    the device: the batched 4x4 kernel for the Kearsley form at the reference tolerances,
    a general n x n kernel (n <= 48, any tol / max_sweeps) otherwise.  Returns ascending
    eigenvalues and sign-normalised eigenvector columns; ValueError for a non-symmetric
    input and RuntimeError when the sweeps do not converge, as the reference."""
    a = np.array(mat, dtype=float)
    n = a.shape[0]
    if a.ndim != 2 or a.shape != (n, n) or not np.allclose(a, a.T, atol=1e-12 * max(1.0, np.abs(a).max())):
        raise ValueError("jacobi_eigh expects a symmetric square matrix")
    if n == 4 and tol == 1e-14 and max_sweeps == 60:
        vals, vecs, flags = K.jacobi4(torch.from_numpy(a.reshape(1, 16)).to(_device()))
    elif 1 <= n <= 48:
        vals, vecs, flags = K.jacobi_n(torch.from_numpy(a.reshape(1, n, n)).to(_device()), tol, max_sweeps)
    else:
        raise ConfigError("device jacobi_eigh supports matrices up to 48 x 48")
    if int(flags.item()) & FLAG_NO_CONVERGE:
        raise RuntimeError("Jacobi diagonalisation did not converge")
    return vals[0].cpu().numpy(), vecs[0].cpu().numpy()


def kearsley_fit_batch(x, a, w, with_derivatives=False):
    """Batched kearsley_fit on device tensors.

    x, a: [B, n, 3] (fitted, reference; used as given, like geometry.py:231);
    w: [n] displacement weights of x (normalised).  Returns a dict of device
    tensors: eig [B,20] (eigvals + row-major eigvectors), quat [B,4], rot
    [B,3,3], flags [B], and rot_grad [B,n,3,3,3] if requested.
    """
    dev = x.device
    B, n, _ = x.shape
    wd = w if (torch.is_tensor(w) and w.shape[0] == K.npad_for(n)) else _wdev(
        w.cpu().numpy() if torch.is_tensor(w) else w, n, dev)
    xc = K.center(x, None, wd, recenter=False)
    ac = K.center(a, None, wd, recenter=False)
    S = K.cov_pairs(xc.planes, ac.planes, None, None, xc.npad, wd)
    eig, quat, rot, flags = K.fit_full(S, xc.g, ac.g)
    out = {"eig": eig, "quat": quat, "rot": rot.reshape(B, 3, 3), "flags": flags}
    if with_derivatives:
        out["rot_grad"] = K.rot_grad(xc.planes, ac.planes, n, xc.npad, wd, eig)
    return out


def kearsley_fit(x: Structure, a: Structure, with_derivatives: bool = False) -> RotationFit:
    """Optimal proper rotation mapping reference ``a`` onto ``x`` (geometry.py:227-263),
    weights = x's displacement weights; DegenerateFitError when derivatives are
    requested and eigvals[1] - eigvals[0] < 1e-9."""
    if x.n_atoms != a.n_atoms:
        raise InvalidStructureError(f"atom count mismatch: {x.n_atoms} vs {a.n_atoms}")
    dev = _device()
    xt = torch.from_numpy(x.coords)[None].to(dev)
    at = torch.from_numpy(a.coords)[None].to(dev)
    res = kearsley_fit_batch(xt, at, x.disp_weights, with_derivatives=False)
    f = int(res["flags"].item())
    eig = res["eig"][0].cpu().numpy()
    eigvals = eig[:4].copy()
    if f & FLAG_NO_CONVERGE:
        raise RuntimeError("Jacobi diagonalisation did not converge")
    rot_grad = None
    if with_derivatives:
        if f & FLAG_DEGENERATE:
            gap = eigvals[1] - eigvals[0]
            raise DegenerateFitError(
                f"eigenvalue gap {gap:.3e} below {DEGENERACY_TOL:.0e}; rotation derivative is ill-defined")
        wd = _wdev(x.disp_weights, x.n_atoms, dev)
        xc = K.center(xt, None, wd, recenter=False)
        ac = K.center(at, None, wd, recenter=False)
        rot_grad = K.rot_grad(xc.planes, ac.planes, x.n_atoms, xc.npad, wd, res["eig"])[0].cpu().numpy()
    return RotationFit(rot=res["rot"][0].cpu().numpy(), quat=res["quat"][0].cpu().numpy(), eigvals=eigvals,
                       rot_grad=rot_grad)


def rotation_derivative_check(x: Structure, a: Structure, h: float = 1e-6) -> float:
    """Analytic dR/dx vs central differences (geometry.py:266-285): all 6n
    bumped fits run as one batched device call."""
    fit = kearsley_fit(x, a, with_derivatives=True)
    n = x.n_atoms
    base = np.repeat(x.coords[None], 6 * n, axis=0)
    idx = np.arange(3 * n)
    base[2 * idx, idx // 3, idx % 3] += h
    base[2 * idx + 1, idx // 3, idx % 3] -= h
    dev = _device()
    res = kearsley_fit_batch(torch.from_numpy(base).to(dev),
                             torch.from_numpy(np.repeat(a.coords[None], 6 * n, axis=0)).to(dev),
                             x.disp_weights)
    rots = res["rot"].cpu().numpy()
    fd = (rots[0::2] - rots[1::2]) / (2.0 * h)
    worst = float(np.abs(fd - fit.rot_grad.reshape(3 * n, 3, 3)).max())
    return worst / max(1.0, float(np.abs(fit.rot_grad).max()))
