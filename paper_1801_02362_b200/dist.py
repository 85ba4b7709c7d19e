"""Multi-GPU plumbing (one process per GPU, torch.distributed; NCCL on GPUs,
gloo for the CPU tests).

Frame sharding (default for configs 2-4): frames are independent objects, so
each rank takes a contiguous slice (``shard_range``) and needs no data-path
collective; results stay on their rank (``gather_frames`` is only for callers
that want them on rank 0).

Landmark sharding (the north_star's variant, ``--shard landmarks``): rank g
owns landmarks [gL/G, (g+1)L/G) and computes, for every frame, the path-CV of
its own shard: s_g, z_g and their gradients.  Because
  Z_g = sum_{i in g} e^{-lam D_i} = e^{-lam z_g}  and  s_g = sum q_i e^{..} / Z_g,
the global values follow from the per-frame pairs (s_g, z_g) alone:
  w_g = Z_g / Z,   s = sum_g w_g s_g,   z = -(1/lam) ln sum_g e^{-lam z_g},
  dz = sum_g w_g dz_g,   ds = sum_g w_g [ds_g - lam (s_g - s) dz_g].
``merge_landmark_shards`` all-gathers the [T, 2] partials (16 B per frame per
rank) and merges them in fixed rank order (bitwise independent of timing);
the gradient combination is an all-reduce of the weighted per-rank
gradients (the one large exchange of this variant).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total, rank, world):
    """Contiguous, balanced [offset, offset + count) of ``total`` items for ``rank``."""
    base, extra = divmod(int(total), int(world))
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count


def merge_partials(s_parts, z_parts, lam):
    """Merge per-shard (s_g, z_g) [G, T] into global (s, z, w [G, T]); fixed order."""
    zmin = torch.min(z_parts, dim=0).values
    e = torch.exp(-lam * (z_parts - zmin[None, :]))
    tot = e.sum(dim=0)
    w = e / tot[None, :]
    s = (w * s_parts).sum(dim=0)
    z = zmin - torch.log(tot) / lam
    return s, z, w


def merge_landmark_shards(s_loc, z_loc, lam, ds_loc=None, dz_loc=None, group=None):
    """All-gather the local (s, z) of this rank's landmark shard and return the
    global (s, z[, ds, dz]).  s_loc, z_loc: [T]; ds_loc, dz_loc: [T, n, 3]."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    local = torch.stack([s_loc, z_loc]).contiguous()
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    P = torch.stack(parts)  # [G, 2, T]
    s, z, w = merge_partials(P[:, 0], P[:, 1], lam)
    if ds_loc is None:
        return s, z
    wg = w[rank][:, None, None]
    ds = wg * (ds_loc - lam * (s_loc - s)[:, None, None] * dz_loc)
    dz = wg * dz_loc
    dist.all_reduce(ds, group=group)
    dist.all_reduce(dz, group=group)
    return s, z, ds, dz


def gather_frames(x, total, group=None):
    """Concatenate frame-sharded per-rank results [count_r, ...] on every rank."""
    world = dist.get_world_size(group)
    sizes = [shard_range(total, r, world)[1] for r in range(world)]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, sizes)])
