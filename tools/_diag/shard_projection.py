"""Landmark-sharded config 4 on ONE GPU: the device time of every rank's share of a
step at G = 1, 2, 4, 8 -- a PROJECTION of the strong-scaling run, not a multi-GPU
measurement.  Each shard engine runs PathCVTC.sharded_steps alone with a replay
"communicator" that answers the two all-reduce-MIN collectives with the global
values (from an unsharded pass over all landmarks), the all-gather with this
shard's own partials repeated (same arithmetic cost), and the all-to-all with no
data movement.  Reports per G: the slowest rank's device time, the mean, the
projected speed-up over G = 1, and the bytes the straddling-row all-to-all would
move (rows with a non-empty window on a non-owner shard x n x 3 x 4 B x 2 CVs).

    python tools/_diag/shard_projection.py [--frames 131072] [--gpus 1,2,4,8]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import dist as D, engine, kernels as K, synth  # noqa: E402


class ReplayComm:
    def __init__(self, dub, dref, world, prune):
        self.answers = [dub, dref] if prune else [dref]  # the order sharded_steps asks in
        self.world = world

    def min(self, t):
        return torch.minimum(self.answers.pop(0).to(t.dtype), t)

    def gather(self, t):
        return torch.stack([t] * self.world)

    def exchange(self, ds, dz, z_parts):
        return torch.zeros(z_parts.shape[1], dtype=torch.int64, device=ds.device)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=131072)
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--balanced", type=int, default=1, help="work-balanced contiguous shards (sample of 8192 frames)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    wl = synth.interp_config_device(41, a.frames, 8192, 10000, 32, dev)
    lms = torch.from_numpy(wl.landmarks).to(dev)
    full = engine.PathCVTC(lms, wl.lam, wl.q)
    fr = wl.frames
    # global per-frame values the two MIN collectives would return
    fr0, fs0 = full._frames(fr, 1, check=False)
    Dc = K.msd_estimate(fs0, full.ls_coarse)
    dub = K.screen_bound(Dc, fs0.opnorm, full.ls_coarse.opnorm, full.kacc, fs0.rnorm, full.ls_coarse.rnorm)
    Dest, _, fss, _, rlo, rhi, perm0 = full._pruned_estimate(fr)
    _, _, dmin, _ = K.candidates(Dest, full.lam, full.cutoff + full.margin, 1, fnorm=full.frame_bound(fss),
                                 fcoef=2.0 * full.lam, rlo=rlo, rhi=rhi)
    dref = torch.empty_like(dmin)
    dref[perm0.long()] = dmin
    load = full.landmark_load(fr[:8192]) if a.balanced else None
    del Dc, Dest, fss, fs0, fr0, full
    torch.cuda.empty_cache()
    base = None
    for G in [int(g) for g in a.gpus.split(",")]:
        times, active = [], 0
        for g in range(G):
            bounds = D.balanced_bounds(load, G) if load is not None else None
            eng = engine.PathCVTC(lms, wl.lam, wl.q, shard=(g, G, bounds))
            for rep in range(2):  # warm-up + timed
                comm = ReplayComm(dub.clone(), dref.clone(), G, eng.prune)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                out = D.drive(eng.sharded_steps(fr), comm)
                e1.record()
                torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            active += int((out["window_cnt"] > 0).sum().item())
            del out, eng
            torch.cuda.empty_cache()
        slow = max(times)
        base = base or slow
        rows = active - a.frames
        print(json.dumps({"G": G, "frames": a.frames, "bounds": bounds, "rank_ms": times,
                          "max_rank_ms": slow, "mean_rank_ms": sum(times) / G,
                          "projected_speedup_vs_G1": base / slow, "projected_frames_per_s": a.frames / slow * 1e3,
                          "straddling_rows": rows, "alltoall_bytes_total": rows * 10000 * 3 * 4 * 2,
                          "note": "projection: per-rank device time on one GPU; collectives not executed"}),
              flush=True)


if __name__ == "__main__":
    main()
