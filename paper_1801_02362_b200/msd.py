"""Drop-in mirror of the SPEC msd-engine module:
DistanceResult, CloseStructureState, exact_distance (Eq. 3/4),
approx_distance (Eq. 5/6), step_close_structure (Alg. 2), step_original
(Alg. 1).  The per-step state machine (counters, the eps test, y <- x) is
host control flow exactly as the SPEC states it; every distance, rotation,
spectrum and gradient is computed by libmcb200 (batched over the reference
set in one launch per kernel).  For whole trajectories use
engine.PathCV.close_replay, which also moves the decisions on device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from ._lib import FLAG_DEGENERATE, call, ptr, stream_ptr
from .colvar import ReferenceSet
from .errors import ConfigError, DegenerateFitError
from .geometry import RotationFit, Structure

I32 = torch.int32


@dataclass
class DistanceResult:
    """value (nm^2), grad dD/dx_k [n, 3], exact (Eq. 3/4) or not (Eq. 5/6) — SPEC.md:100-104."""

    value: float
    grad: np.ndarray
    exact: bool


@dataclass
class CloseStructureState:
    """close structure y, fit x<->y, saved R_{a_i y}, eps and counters."""

    epsilon: float = 0.01  # nm^2, PAPER.md computational details / SPEC.md:161
    y: Structure | None = None
    fit_xy: RotationFit | None = None
    saved_rots: np.ndarray | None = None
    reassign_count: int = 0
    step_count: int = 0
    expensive_count: int = 0
    cheap_count: int = 0
    _xy_eig: np.ndarray | None = field(default=None, repr=False)

    def __post_init__(self):
        if not (self.epsilon >= 0):
            raise ConfigError("epsilon must be >= 0")


def _dev():
    K.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _frames(structs, refd):
    coords = torch.from_numpy(np.stack([s.coords for s in structs])).to(_dev())
    return K.center(coords, refd["wa"], refd["w"])


def _exact_batch(x: Structure, ref: ReferenceSet, indices):
    """Exact D, R and Eq. 4 gradients of x against ref.structures[indices]."""
    refd = ref.device(x.disp_weights, x.align_weights)
    lm = refd["c"]
    fr = _frames([x], refd)
    S = K.cov_dense(fr, lm)  # [1, N, 9]
    D, R, _, flags = K.fit_dense(S, fr.g, lm.g, want_rot=True)
    idx = torch.as_tensor(np.asarray(indices, dtype=np.int32), device=fr.planes.device)
    P = int(idx.shape[0])
    xi = torch.zeros(P, dtype=I32, device=idx.device)
    rot = R[0].index_select(0, idx.long()).contiguous()
    grad = torch.empty((P, x.n_atoms, 3), dtype=torch.float64, device=idx.device)
    call("mc_pair_grad", P, x.n_atoms, fr.npad, ptr(fr.planes), ptr(lm.planes), ptr(xi), ptr(idx), ptr(rot),
         ptr(refd["w"]), ptr(refd["wa"]), ptr(fr.wbar), ptr(lm.wbar), None, None, None, None, None, None, None,
         None, None, ptr(grad), stream_ptr())
    D = D[0].index_select(0, idx.long())
    return D.cpu().numpy(), rot.reshape(P, 3, 3).cpu().numpy(), grad.cpu().numpy()


def _approx_batch(x: Structure, state: CloseStructureState, ref: ReferenceSet, indices):
    refd = ref.device(x.disp_weights, x.align_weights)
    lm = refd["c"]
    fr = _frames([x, state.y], refd)  # frame 0 = x, frame 1 = y
    dev = fr.planes.device
    idx = torch.as_tensor(np.asarray(indices, dtype=np.int32), device=dev)
    P = int(idx.shape[0])
    xi = torch.zeros(P, dtype=I32, device=dev)
    yi = torch.ones(P, dtype=I32, device=dev)
    approx = torch.ones(P, dtype=I32, device=dev)
    S = K.cov_pairs(fr.planes, lm.planes, xi, idx, fr.npad, refd["w"])
    rot = torch.from_numpy(np.ascontiguousarray(state.saved_rots[np.asarray(indices)].reshape(P, 9))).to(dev)
    eig = torch.from_numpy(np.repeat(state._xy_eig[None], P, axis=0)).to(dev)
    rxy = torch.from_numpy(np.repeat(state.fit_xy.rot.reshape(1, 9), P, axis=0)).to(dev)
    value = torch.empty(P, dtype=torch.float64, device=dev)
    grad = torch.empty((P, x.n_atoms, 3), dtype=torch.float64, device=dev)
    call("mc_pair_grad", P, x.n_atoms, fr.npad, ptr(fr.planes), ptr(lm.planes), ptr(xi), ptr(idx), ptr(rot),
         ptr(refd["w"]), ptr(refd["wa"]), ptr(fr.wbar), ptr(lm.wbar), ptr(approx), ptr(yi), ptr(S), ptr(lm.mom),
         ptr(eig), ptr(rxy), ptr(fr.g), ptr(lm.g), ptr(value), ptr(grad), stream_ptr())
    return value.cpu().numpy(), grad.cpu().numpy()


def exact_distance(x: Structure, a: Structure, state: CloseStructureState | None = None) -> DistanceResult:
    """Eq. 3/4: D = sum w |x - R a|^2 and dD/dx (raw coords);
    increments state.expensive_count when a state is supplied."""
    ref = ReferenceSet([a], lam=1.0)
    D, _, g = _exact_batch(x, ref, [0])
    if state is not None:
        state.expensive_count += 1
    return DistanceResult(float(D[0]), g[0], True)


def approx_distance(x: Structure, a_index: int, state: CloseStructureState, ref: ReferenceSet) -> DistanceResult:
    """Eq. 5/6 with the state's R_xy (and its dR/dx) and saved R_{a y}."""
    if state.y is None or state.saved_rots is None or state.fit_xy is None or state._xy_eig is None:
        raise ConfigError("approx_distance needs a state with a close structure and a current x<->y fit")
    if not (0 <= a_index < ref.n):
        raise ConfigError("reference index out of range")
    v, g = _approx_batch(x, state, ref, [a_index])
    state.cheap_count += 1
    return DistanceResult(float(v[0]), g[0], False)


def _fit_xy(x: Structure, y: Structure):
    from .geometry import kearsley_fit_batch

    dev = _dev()
    xt = torch.from_numpy(x.center().coords)[None].to(dev)
    yt = torch.from_numpy(y.coords)[None].to(dev)
    res = kearsley_fit_batch(xt, yt, x.disp_weights)
    eig = res["eig"][0].cpu().numpy()
    fit = RotationFit(rot=res["rot"][0].cpu().numpy(), quat=res["quat"][0].cpu().numpy(), eigvals=eig[:4].copy())
    return fit, eig, int(res["flags"].item())


def step_close_structure(x: Structure, state: CloseStructureState, ref: ReferenceSet):
    """Alg. 2 lines 2-17: returns (state, [DistanceResult] * N)."""
    state.step_count += 1
    state.expensive_count += 1  # D(x, y) is always computed
    if state.y is None:
        refresh = True
        state.fit_xy, state._xy_eig = None, None
    else:
        fit, eig, flags = _fit_xy(x, state.y)
        if flags & FLAG_DEGENERATE:
            raise DegenerateFitError("x<->y fit has a degenerate spectrum; dR_xy/dx is ill-defined")
        state.fit_xy, state._xy_eig = fit, eig
        refresh = bool(fit.eigvals[0] > state.epsilon)  # strict
    all_idx = list(range(ref.n))
    if refresh:
        D, R, g = _exact_batch(x, ref, all_idx)
        state.y = x.center()
        state.saved_rots = R
        # the state now describes x against its own close structure: R_xy = I with
        # x's spectrum, so approx_distance right after a reassignment equals the
        # exact distance instead of reusing the fit to the old y
        state.fit_xy, state._xy_eig, _ = _fit_xy(x, state.y)
        state.reassign_count += 1
        state.expensive_count += ref.n
        return state, [DistanceResult(float(D[i]), g[i], True) for i in all_idx]
    v, g = _approx_batch(x, state, ref, all_idx)
    state.cheap_count += ref.n
    return state, [DistanceResult(float(v[i]), g[i], False) for i in all_idx]


def step_original(x: Structure, nl, ref: ReferenceSet, state: CloseStructureState | None = None):
    """Alg. 1: exact distances to the neighbour-list members
    (``nl`` = iterable of indices, or None for all references)."""
    idx = list(range(ref.n)) if nl is None else sorted(int(i) for i in (nl.indices if hasattr(nl, "indices") else nl))
    D, _, g = _exact_batch(x, ref, idx)
    if state is not None:
        state.expensive_count += len(idx)
        state.step_count += 1
    return [(i, DistanceResult(float(D[k]), g[k], True)) for k, i in enumerate(idx)]
