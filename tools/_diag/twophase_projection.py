"""Two-phase landmark-sharded config 4 on ONE GPU: the device time of every rank's share
of a step at G = 1, 2, 4, 8 -- a PROJECTION of the strong-scaling run, not a multi-GPU
measurement (this pool gives one GPU).  Rank g of G runs PathCVTC.two_phase_steps on its
T/G home frames with a replay communicator whose answers come from an unsharded pass:
the all-gathered screening operand of all T frames (split once, outside the timed
region: on hardware it arrives over NVLink), the global D_min bound and estimate minimum
(the two all-reduce MINs), and the unsharded windows for the all-gather of per-shard
windows (their hull is the unsharded window by construction).  Each rank: one warm-up and
three timed runs, the minimum kept.  Reports per G the slowest rank's device time, the
ideal t(1)/G, their ratio, and the NCCL bytes per step.

    python tools/_diag/twophase_projection.py [--frames 131072] [--gpus 1,2,4,8]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import dist as D, engine, kernels as K, synth  # noqa: E402


class RoutedReplayComm:
    """Answers of the routed phase 1 for rank g: the counts, the frames whose global hull
    meets shard g (from every home rank: rows of the all-frames split), the global estimate
    minimum, and the unsharded windows of the home frames it sent."""

    def __init__(self, counts, recv, dref, win):
        self.counts, self.recv, self.dref, self.win = counts, recv, dref, win
        self.sent = None

    def gather(self, t):
        return torch.tensor(self.counts, dtype=torch.int64, device=t.device)[:, None]

    def alltoallv(self, fields):
        if self.sent is None:  # the operand rows: what shard g receives from every home
            self.sent = [b.long() for b in fields[0]]
            return [[x] for x in self.recv]
        # the windows: shard r's windows of the frames sent to r (their hull = unsharded)
        return [[self.win[:, ids].T.contiguous().to(torch.int32) for ids in self.sent]]

    def min(self, t):
        return torch.minimum(self.dref.to(t.dtype), t)


class ReplayComm:
    def __init__(self, fs_all, counts, dub, dref, win):
        self.fs_all, self.counts = fs_all, counts
        self.mins = [dub, dref]
        self.win = win

    def allgather_split(self, sp):
        return self.fs_all, self.counts

    def min(self, t):
        return torch.minimum(self.mins.pop(0).to(t.dtype), t)

    def gather(self, t):
        return self.win[None]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=131072)
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--routed", type=int, default=0, help="routed phase 1 (PathCVTC(route=True, two_phase=True))")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    wl = synth.interp_config_device(41, a.frames, 8192, 10000, 32, dev)
    lms = torch.from_numpy(wl.landmarks).to(dev)
    full = engine.PathCVTC(lms, wl.lam, wl.q)
    fr = wl.frames
    T = fr.shape[0]
    fr0, fs0 = full._frames(fr, 1, check=False)
    Dc = K.msd_estimate(fs0, full.ls_coarse)
    dub = K.screen_bound(Dc, fs0.opnorm, full.ls_coarse.opnorm, full.kacc, fs0.rnorm, full.ls_coarse.rnorm)
    Dest, _, fss, _, rlo, rhi, perm0 = full._pruned_estimate(fr)
    _, _, dmin, _ = K.candidates(Dest, full.lam, full.cutoff + full.margin, 1, fnorm=full.frame_bound(fss),
                                 fcoef=2.0 * full.lam, rlo=rlo, rhi=rhi)
    dref = torch.empty_like(dmin)
    dref[perm0.long()] = dmin
    ref = full.evaluate(fr, grad=False)
    win = torch.stack([ref["window_lo"], ref["window_cnt"]]).to(torch.int32)
    if a.routed:  # every frame's global coarse hull (what the home ranks route on)
        hlo_g, hhi_g, _ = K.prune_plan(Dc, fs0.opnorm, full.ls_coarse.opnorm, full.kacc, full.mind,
                                       (full.cutoff + 2.0) / full.lam, full.knear, maxd=full.maxd,
                                       cstride=full.cstride, frnorm=fs0.rnorm, crnorm=full.ls_coarse.rnorm)
    del Dc, Dest, fss, full, ref
    torch.cuda.empty_cache()
    opbytes = fs0.hi.numel() * fs0.hi.element_size() + T * 8 * 7  # halves + per-frame scalars
    rows = []
    base = None
    for G in [int(g) for g in a.gpus.split(",")]:
        times, recv_frames = [], []
        counts = [D.shard_range(T, g, G)[1] for g in range(G)]
        tbounds = D.tile_bounds(8192, G)
        for g in range(G):
            off, cnt = D.shard_range(T, g, G)
            if a.routed:
                eng = engine.PathCVTC(lms, wl.lam, wl.q, shard=(g, G, tbounds), route=True, two_phase=True)
                t0, t1 = tbounds[g] // 48, (tbounds[g + 1] + 47) // 48
                ids = torch.nonzero((hlo_g < t1) & (hhi_g > t0)).flatten()
                recv = [ids, *[fs0.hi[pl, ids].contiguous() for pl in range(3)],
                        torch.stack([fs0.scale[ids], fs0.opnorm[ids], fs0.rnorm[ids], fs0.g[ids]], 1),
                        torch.stack([hlo_g[ids], hhi_g[ids]], 1)]
                recvd = int(ids.numel())
            else:
                eng = engine.PathCVTC(lms, wl.lam, wl.q, shard=(g, G), two_phase=True)
                recvd = T
            home = fr[off:off + cnt]
            best = float("inf")
            for rep in range(4):  # warm-up + 3 timed; the minimum (allocator / clock transients
                # of a rank timed alone land on single runs)
                comm = (RoutedReplayComm(counts, recv, dref.clone(), win) if a.routed else
                        ReplayComm(fs0, counts, dub.clone(), dref.clone(), win))
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                out = D.drive(eng.two_phase_steps(home, off, T, grad=True), comm)
                e1.record()
                torch.cuda.synchronize()
                if rep:
                    best = min(best, e0.elapsed_time(e1))
            times.append(best)
            recv_frames.append(recvd)
            if g == G - 1 and os.environ.get("PROJ_KERNELS"):  # per-kernel breakdown of one rank
                from paper_1801_02362_b200 import _lib
                comm = (RoutedReplayComm(counts, recv, dref.clone(), win) if a.routed else
                        ReplayComm(fs0, counts, dub.clone(), dref.clone(), win))
                _lib.start_profile()
                torch.cuda.synchronize()
                e0.record()
                D.drive(eng.two_phase_steps(home, off, T, grad=True), comm)
                e1.record()
                prof = _lib.stop_profile()
                kt = sum(t for _, t in prof.values())
                print(json.dumps({"G": G, "rank": g, "total_ms": e0.elapsed_time(e1), "library_kernels_ms": kt,
                                  "kernels": {k: round(t, 3) for k, (c, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])}}),
                      file=sys.stderr, flush=True)
            del out, eng
            torch.cuda.empty_cache()
        slow = max(times)
        base = slow if G == 1 else base
        ideal = base / G
        # NCCL per step: all-gather of the screening operand (each rank receives the others'
        # home frames), two all-reduce MINs (T x 8 B, T x 4 B), all-gather of windows (G x 2 x T x 4 B)
        if a.routed:  # each rank receives the frames whose hull meets its shard, (G-1)/G of them remote
            recv = max(recv_frames) * (opbytes / T) * (G - 1) / G
            nccl = {"alltoallv_operand_recv_max": recv, "allreduce_min": 4 * T, "alltoallv_windows": 8 * max(recv_frames)}
        else:
            recv = opbytes * (G - 1) / G
            nccl = {"allgather_split_recv": recv, "allreduce_min": 12 * T, "allgather_windows": 8 * T * G}
        row = {"G": G, "routed": bool(a.routed), "slowest_rank_ms": slow, "mean_rank_ms": sum(times) / G,
               "ideal_ms": ideal, "slowest_over_ideal": slow / ideal, "projected_speedup": base / slow,
               "nccl_bytes_per_rank": nccl, "operand_recv_ms_at_700GBps": recv / 700e9 * 1e3,
               "received_frames": recv_frames, "rank_ms": times, "frames": T}
        rows.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
