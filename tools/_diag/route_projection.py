"""Frame-routed landmark sharding (PathCVTC(..., route=True)) of config 4 at G = 1, 2,
4, 8, all ranks emulated on ONE GPU in lock step (dist.drive_lockstep semantics): each
rank's generator segments are timed with CUDA events (per-rank device time of a step),
collectives are computed locally and their payload bytes counted.  A PROJECTION of the
strong-scaling run, not a multi-GPU measurement: the projected step is the slowest
rank's time (+ the all-to-all bytes / NVLink bandwidth, reported separately).

    python tools/_diag/route_projection.py [--frames 131072] [--gpus 1,2,4,8]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import dist as D, engine, synth  # noqa: E402


def timed_lockstep(gens):
    G = len(gens)
    ms = [0.0] * G
    seg = [[] for _ in range(G)]
    nbytes = 0

    def step(i, val):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            r = next(gens[i]) if val is None else gens[i].send(val)
            done = None
        except StopIteration as e:
            r, done = None, e.value
        e1.record()
        torch.cuda.synchronize()
        ms[i] += e0.elapsed_time(e1)
        seg[i].append(round(e0.elapsed_time(e1), 2))
        return r, done

    reqs, results = [None] * G, [None] * G
    for i in range(G):
        reqs[i], _ = step(i, None)
    while True:
        op = reqs[0][0]
        if op == "min":
            v = torch.stack([r[1] for r in reqs]).amin(0)
            outs = [v.clone() for _ in range(G)]
        elif op == "gather":
            v = torch.stack([r[1] for r in reqs])
            outs = [v for _ in range(G)]
            nbytes += v.numel() * v.element_size()
        elif op == "alltoallv":
            nf = len(reqs[0][1])
            outs = [[[reqs[g][1][f][h] for g in range(G)] for f in range(nf)] for h in range(G)]
            for g in range(G):
                for f in range(nf):
                    for h in range(G):
                        if h != g:
                            b = reqs[g][1][f][h]
                            nbytes += b.numel() * b.element_size()
        else:
            raise RuntimeError(op)
        for i in range(G):
            reqs[i], done = step(i, outs[i])
            if done is not None:
                results[i] = done
        if all(r is not None for r in results):
            timed_lockstep.segments = seg
            return results, ms, nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=131072)
    ap.add_argument("--gpus", default="1,2,4,8")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    wl = synth.interp_config_device(41, a.frames, 8192, 10000, 32, dev)
    lms = torch.from_numpy(wl.landmarks).to(dev)
    base = None
    for G in [int(g) for g in a.gpus.split(",")]:
        b = D.tile_bounds(8192, G)
        engs = [engine.PathCVTC(lms, wl.lam, wl.q, shard=(g, G, b), route=True) for g in range(G)]
        for rep in range(2):  # warm-up + timed
            gens = []
            for g, e in enumerate(engs):
                off, cnt = D.shard_range(a.frames, g, G)
                gens.append(e.routed_steps(wl.frames[off:off + cnt], off, a.frames))
            outs, ms, nbytes = timed_lockstep(gens)
            recv = [o["received"] for o in outs]
            del outs, gens
            torch.cuda.empty_cache()
        slow = max(ms)
        base = base or slow
        print(json.dumps({"G": G, "frames": a.frames, "bounds": b, "rank_ms": ms, "max_rank_ms": slow,
                          "mean_rank_ms": sum(ms) / G, "projected_speedup_vs_G1": base / slow,
                          "projected_frames_per_s": a.frames / slow * 1e3, "frames_received": recv,
                          "exchange_bytes_total": nbytes, "segments_ms": timed_lockstep.segments,
                          "exchange_ms_at_700GBps_per_gpu": nbytes / G / 700e9 * 1e3,
                          "note": "projection: per-rank device time emulated on one GPU; collectives not executed"}),
              flush=True)
        del engs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
