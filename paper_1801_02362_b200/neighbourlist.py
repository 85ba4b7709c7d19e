"""Neighbour list (SPEC [MODULE] neighbourlist).

Mirror of the spec's ``NeighbourList`` type and ``maybe_update`` operation:
the M closest reference structures, refreshed every ``stride`` steps from the
distances to ALL references (exact in original mode, the approximated ones in
close-structure mode).  Selection runs on the device (``mc_neighbour_topm``):
indices of the M smallest distances, ties broken by the lower index, kept in
ascending order.  Batched use (one list per frame / walker) goes through
``kernels.neighbour_topm`` and ``PathCV.close_replay(neighbours=M, nl_stride=...)``.
"""

from __future__ import annotations

import torch

from . import kernels as K
from .errors import ConfigError


class NeighbourList:
    """indices: int32 CUDA tensor [M] (ascending); size M; stride >= 1;
    last_update_step (None before the first update); enabled.

    A disabled list behaves as M = N, stride = 1 (every reference active,
    SPEC "Invariants & Properties")."""

    def __init__(self, n_refs, size, stride=1, enabled=True, device=None):
        if not enabled:
            size, stride = n_refs, 1
        if not 1 <= int(size) <= int(n_refs):
            raise ConfigError("neighbour list size must satisfy 1 <= M <= N")  # SPEC: M > N -> configuration error
        if int(stride) < 1:
            raise ConfigError("neighbour list stride must be >= 1")
        self.n_refs, self.size, self.stride, self.enabled = int(n_refs), int(size), int(stride), bool(enabled)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.indices = torch.arange(self.size, dtype=torch.int32, device=self.device)
        self.last_update_step = None

    def due(self, step):
        return self.last_update_step is None or step - self.last_update_step >= self.stride

    def maybe_update(self, step, distances_all):
        """Update from the distances to all N references if ``step`` is due; returns self."""
        if not self.due(step):
            return self
        d = torch.as_tensor(distances_all)
        if d.ndim != 1 or d.shape[0] != self.n_refs:
            raise ConfigError("distances_all must hold one distance per reference")
        if not self.enabled:
            self.indices = torch.arange(self.n_refs, dtype=torch.int32, device=self.device)
        else:
            d = d.to(device=self.device)
            if d.dtype not in (torch.float32, torch.float64):
                d = d.double()
            self.indices = K.neighbour_topm(d.reshape(1, -1).contiguous(), self.size)[0]
        self.last_update_step = int(step)
        return self
