"""Multi-GPU plumbing (one process per GPU, torch.distributed; NCCL on GPUs,
gloo for the CPU tests).

Frame sharding (default for configs 2-4): frames are independent objects, so
each rank takes a contiguous slice (``shard_range``) and needs no data-path
collective; results stay on their rank (``gather_frames`` is only for callers
that want them on rank 0).

Landmark sharding (the north_star's variant, ``bench.py --shard landmarks``,
``PathCVTC(..., shard=(rank, world))``): rank g owns landmarks
[gL/G, (g+1)L/G) and every frame.  Per-frame exchanges, all O(T):
  1. all-reduce MIN of the coarse screen's D_min upper bound (pruning) and of the
     screen estimate's minimum -- every shard takes its windows against the global
     minimum, so a shard far from a frame computes nothing for it;
  2. all-gather of the per-frame partials (s_g, z_g) of each shard's exact window
     (16 B per frame per rank).  Because
       Z_g = sum_{i in g} e^{-lam D_i} = e^{-lam z_g}  and  s_g = sum q_i e^{..} / Z_g,
     the global values follow from them alone (``merge_partials``, fixed rank order,
     bitwise independent of timing):
       w_g = Z_g / Z,   s = sum_g w_g s_g,   z = -(1/lam) ln sum_g e^{-lam z_g},
       dz = sum_g w_g dz_g,   ds = sum_g w_g [ds_g - lam (s_g - s) dz_g];
     each shard rescales its coefficients by (alpha, beta) = (w_g, -lam (s_g - s))
     on the device (mc_shard_rescale) before its gradient pass;
  3. the gradient rows: frame t is owned by the shard with the largest Z_g (its
     nearest landmark); shards whose window of t is non-empty but that do not own
     it send their rows to the owner (one all-to-all of the straddling rows only,
     ``exchange_owned_rows``).  The dense alternative, an all-reduce of T x n x 3
     per CV (``merge_landmark_shards``), moves 31 GB per step at config 4.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(total, rank, world):
    """Contiguous, balanced [offset, offset + count) of ``total`` items for ``rank``."""
    base, extra = divmod(int(total), int(world))
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count


def balanced_bounds(load, world, floor=1.0):
    """Contiguous landmark shards with equal work: cut the cumulative per-landmark load
    (``PathCVTC.landmark_load`` on a frame sample, plus ``floor`` per landmark for the
    per-landmark fixed costs) at its G quantiles.  Returns G + 1 offsets 0 = b_0 < ... <
    b_G = L (every shard keeps >= 1 landmark)."""
    load = torch.as_tensor(load, dtype=torch.float64).cpu() + float(floor)
    L = int(load.numel())
    if not 1 <= world <= L:
        raise ValueError("1 <= world <= number of landmarks")
    cum = torch.cumsum(load, 0)
    tot = float(cum[-1])
    b = [0]
    for g in range(1, world):
        cut = int(torch.searchsorted(cum, torch.tensor(tot * g / world, dtype=torch.float64)).item()) + 1
        b.append(min(max(cut, b[-1] + 1), L - (world - g)))
    b.append(L)
    return b


def tile_bounds(L, world, load=None, tile=48):
    """Contiguous landmark shards cut at multiples of the screen's 48-landmark tile (the
    frame-routed variant routes frames by tile hulls): balanced by ``load`` (per-landmark
    work, ``PathCVTC.landmark_load``) when given, else by landmark count."""
    ntl = (int(L) + tile - 1) // tile
    if not 1 <= world <= ntl:
        raise ValueError("1 <= world <= number of landmark tiles")
    if load is None:
        tl = torch.ones(ntl, dtype=torch.float64)
    else:
        ld = torch.as_tensor(load, dtype=torch.float64).cpu() + 1.0
        tl = torch.nn.functional.pad(ld, (0, ntl * tile - int(L))).view(ntl, tile).sum(1)
    b = balanced_bounds(tl, world, floor=0.0)
    return [min(int(L), x * tile) for x in b]


def merge_partials(s_parts, z_parts, lam):
    """Merge per-shard (s_g, z_g) [G, T] into global (s, z, w [G, T]); fixed order.
    A shard with an empty window for frame t reports z_g = +inf (w_g = 0)."""
    zmin = torch.min(z_parts, dim=0).values
    e = torch.exp(-lam * (z_parts - zmin[None, :]))
    e = torch.where(torch.isinf(z_parts), torch.zeros_like(e), e)
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


# ---------------------------------------------------------------- landmark-sharded exchanges

def shard_coefficients(s_parts, z_parts, lam, rank):
    """Global (s, z) and this shard's coefficient rescaling (alpha, beta) [T]:
    cs' = alpha (cs + beta cz), cz' = alpha cz."""
    s, z, w = merge_partials(s_parts, z_parts, lam)
    alpha = w[rank].contiguous()
    beta = (-lam * (s_parts[rank] - s)).contiguous()
    return s, z, alpha, beta


def gradient_owners(z_parts):
    """Owner shard of every frame: the largest Z_g (smallest z_g; ties to the lower rank)."""
    return torch.argmin(z_parts, dim=0)


def exchange_plan(z_parts, rank):
    """Rows this rank sends to / receives from every other rank: frame t goes from every
    shard with a non-empty window (finite z_g) to its owner."""
    world = z_parts.shape[0]
    owner = gradient_owners(z_parts)
    active = torch.isfinite(z_parts)
    send = [torch.nonzero(active[rank] & (owner == h)).flatten() if h != rank else None for h in range(world)]
    recv = [torch.nonzero(active[g] & (owner == rank)).flatten() if g != rank else None for g in range(world)]
    return owner, send, recv


def _alltoall_rows(bufs_send, recv_counts, row_shape, dtype, device, group=None):
    """Variable-size all-to-all of row blocks (one all_to_all_single on packed buffers)."""
    world = len(bufs_send)
    rowlen = int(np.prod(row_shape)) if row_shape else 1
    send_counts = [0 if b is None else int(b.shape[0]) for b in bufs_send]
    flat = [b.reshape(-1) for b in bufs_send if b is not None and b.shape[0]]
    sendbuf = torch.cat(flat) if flat else torch.empty((0,), dtype=dtype, device=device)
    recvbuf = torch.empty((sum(recv_counts) * rowlen,), dtype=dtype, device=device)
    dist.all_to_all_single(recvbuf, sendbuf, [c * rowlen for c in recv_counts], [c * rowlen for c in send_counts],
                           group=group)
    out, off = [], 0
    for g in range(world):
        c = recv_counts[g]
        out.append(recvbuf[off * rowlen:(off + c) * rowlen].view((c,) + tuple(row_shape)))
        off += c
    return out


def exchange_owned_rows(ds, dz, z_parts, group=None):
    """Complete the gradient rows this rank owns: add the straddling rows of the other
    shards (in fixed rank order).  ds, dz: [T, n, 3] partial sums of this shard.
    Returns owner [T]; rows with owner != rank stay partial and must be ignored."""
    rank = dist.get_rank(group)
    owner, send, recv = exchange_plan(z_parts, rank)
    if len(send) == 1:
        return owner
    row_shape = (2,) + tuple(ds.shape[1:])
    bufs = [None if idx is None else torch.stack([ds[idx], dz[idx]], dim=1) for idx in send]
    counts = [0 if idx is None else int(idx.numel()) for idx in recv]
    got = _alltoall_rows(bufs, counts, row_shape, ds.dtype, ds.device, group)
    for g, idx in enumerate(recv):
        if idx is None or idx.numel() == 0:
            continue
        ds.index_add_(0, idx.to(ds.device), got[g][:, 0])
        dz.index_add_(0, idx.to(dz.device), got[g][:, 1])
    return owner


class DistComm:
    """Collectives of the landmark-sharded evaluation over a torch.distributed group."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def min(self, t):
        t = t.clone()
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return t

    def gather(self, t):
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.stack(parts)

    def exchange(self, ds, dz, z_parts):
        return exchange_owned_rows(ds, dz, z_parts, self.group)

    def allgather_split(self, sp):
        """All-gather of a frame Split (the one-term screening operand + per-frame scalars)
        over the ranks, concatenated in rank order (ragged frame counts); returns
        (Split, per-rank frame counts)."""
        from .kernels import Split

        counts = torch.tensor([sp.count], dtype=torch.int64, device=sp.hi.device)
        allc = self.gather(counts).flatten().cpu().tolist()
        return (concat_splits([_gather_ragged(self, x, allc, dim) for x, dim in _split_fields(sp)], sp, allc, Split),
                allc)

    def alltoallv(self, fields):
        """fields: list of per-destination row blocks (same row counts across fields).
        Returns, per field, the list of blocks received from every source rank."""
        if self.world == 1:
            return [list(blocks) for blocks in fields]
        counts = torch.tensor([int(b.shape[0]) for b in fields[0]], dtype=torch.int64, device=fields[0][0].device)
        rcounts = torch.empty_like(counts)
        dist.all_to_all_single(rcounts, counts, group=self.group)
        rc = rcounts.cpu().tolist()
        out = []
        for blocks in fields:
            shape = tuple(blocks[0].shape[1:])
            out.append(_alltoall_rows([b.contiguous() for b in blocks], rc, shape, blocks[0].dtype,
                                      blocks[0].device, self.group))
        return out


def _split_fields(sp):
    """(tensor, frame dim) of every per-frame field of a Split (None fields skipped later)."""
    return [(sp.hi, 1), (sp.lo, 1), (sp.scale, 0), (sp.opnorm, 0), (sp.rnorm, 0), (sp.centroid, 0), (sp.g, 0),
            (sp.wbar, 0), (sp.mom, 0)]


def _gather_ragged(comm, x, counts, dim):
    """All-gather of [.., count_r, ..] blocks along `dim` (padded to the largest count)."""
    if x is None:
        return None
    mx = max(counts)
    if x.shape[dim] < mx:
        pad_shape = list(x.shape)
        pad_shape[dim] = mx - x.shape[dim]
        x = torch.cat([x, torch.zeros(pad_shape, dtype=x.dtype, device=x.device)], dim=dim)
    parts = comm.gather(x.contiguous())  # [G, ...]
    return torch.cat([parts[r].narrow(dim, 0, c) for r, c in enumerate(counts)], dim=dim)


def concat_splits(fields, like, counts, cls):
    """Assemble the gathered Split (the order of _split_fields)."""
    hi, lo, scale, opnorm, rnorm, centroid, g, wbar, mom = fields
    flags = torch.zeros((sum(counts),), dtype=torch.uint8, device=like.hi.device)
    return cls(hi.contiguous(), None if lo is None else lo.contiguous(), centroid, g, wbar, mom, flags, like.n,
               like.kpad, scale, like.fmt, like.terms, opnorm, rnorm)


def drive(steps, comm):
    """Run a landmark-sharded evaluation generator (PathCVTC.sharded_steps) against
    ``comm``: every yielded (op, *args) is one collective; returns its final value."""
    try:
        req = next(steps)
        while True:
            op, args = req[0], req[1:]
            req = steps.send(getattr(comm, op)(*args))
    except StopIteration as e:
        return e.value


def drive_lockstep(steps_list, lam=None):
    """Run G shard generators in one process, in lock step, with the collectives
    computed locally (the same merge arithmetic as DistComm; one device, no
    inter-rank waits).  Used by the single-GPU tests of the sharded path."""
    G = len(steps_list)
    reqs = [next(g) for g in steps_list]
    results = [None] * G
    while True:
        ops = {r[0] for r in reqs}
        if len(ops) != 1:
            raise RuntimeError(f"shards out of step: {ops}")
        op = ops.pop()
        if op == "min":
            v = torch.stack([r[1] for r in reqs]).amin(0)
            outs = [v.clone() for _ in range(G)]
        elif op == "gather":
            v = torch.stack([r[1] for r in reqs])
            outs = [v for _ in range(G)]
        elif op == "allgather_split":
            from .kernels import Split

            sps = [r[1] for r in reqs]
            counts = [sp.count for sp in sps]
            fields = []
            for k, (_, dim) in enumerate(_split_fields(sps[0])):
                xs = [_split_fields(sp)[k][0] for sp in sps]
                fields.append(None if xs[0] is None else torch.cat(xs, dim=dim))
            v = concat_splits(fields, sps[0], counts, Split)
            outs = [(v, counts) for _ in range(G)]
        elif op == "alltoallv":
            nf = len(reqs[0][1])
            outs = [[[reqs[g][1][f][h] for g in range(G)] for f in range(nf)] for h in range(G)]
        elif op == "exchange":
            # every shard's rows, owner-summed in rank order
            z_parts = reqs[0][3]
            owner, _, _ = exchange_plan(z_parts, 0)
            active = torch.isfinite(z_parts)
            for h in range(G):
                ds_h, dz_h = reqs[h][1], reqs[h][2]
                for g in range(G):
                    if g == h:
                        continue
                    idx = torch.nonzero(active[g] & (owner == h)).flatten()
                    if idx.numel():
                        ds_h.index_add_(0, idx, reqs[g][1][idx])
                        dz_h.index_add_(0, idx, reqs[g][2][idx])
            outs = [owner for _ in range(G)]
        else:
            raise RuntimeError(f"unknown collective {op!r}")
        done = 0
        for i, g in enumerate(steps_list):
            if results[i] is not None:
                continue
            try:
                reqs[i] = g.send(outs[i])
            except StopIteration as e:
                results[i] = e.value
                done += 1
        if all(r is not None for r in results):
            return results
        if done:
            raise RuntimeError("shards finished out of step")
