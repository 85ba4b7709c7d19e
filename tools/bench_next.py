"""Measurement of the §8(f) "next" rows on config-4 shapes (B200):

* neighbour top-M selection (`mc_neighbour_topm`) over a [T, L] fp32 distance
  matrix — HBM-bound: algorithmic bytes = 4 T L read + 4 T M written;
* metadynamics bias force (`mc_mtd_force`) on the path-CV gradients
  [T, N, 3] fp32 (ds, dz) — HBM-bound: 2 x 12 T N read + 12 T N written;
* direct hill sum (`mc_mtd_bias_direct`) for T frames x H hills — one exp per
  (frame, hill): reported as Gexp/s;
* the toy MD driver (`mc_toysim_run`, SPEC toysim, 8(f) 3): W walkers x S steps
  of an 8-bead chain against 16 references in the close-structure and original
  modes, one launch — walker-steps/s, beside the numpy oracle's rate (1 core).

CUDA events, after warm-up; prints one JSON line per kernel with the roofline
fraction against MEASURED_PEAKS.json hbm_gbs.
    python tools/bench_next.py [--T 131072 --L 8192 --N 10000 --M 64 --H 4096]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))

from paper_1801_02362_b200 import _lib, kernels as K  # noqa: E402
from paper_1801_02362_b200.metadynamics import HillStore  # noqa: E402


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=131072)
    ap.add_argument("--L", type=int, default=8192)
    ap.add_argument("--N", type=int, default=10000)
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--W", type=int, default=4096, help="toy MD walkers")
    ap.add_argument("--S", type=int, default=2000, help="toy MD steps per launch")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")) as f:
        hbm = json.load(f)["hbm_gbs"]
    g = torch.Generator(device=dev).manual_seed(0)
    # neighbour top-M
    D = torch.rand((a.T, a.L), generator=g, device=dev)
    ms = timed(lambda: K.neighbour_topm(D, a.M))
    byt = 4.0 * a.T * a.L + 4.0 * a.T * a.M
    print(json.dumps({"kernel": "mc_neighbour_topm", "shape": [a.T, a.L, a.M], "ms": ms,
                      "achieved_GBps": byt / ms / 1e6, "peak_GBps": hbm, "frac": byt / ms / 1e6 / hbm}))
    del D
    # bias force
    ds = torch.randn((a.T, a.N, 3), generator=g, device=dev)
    dz = torch.randn((a.T, a.N, 3), generator=g, device=dev)
    st = HillStore(2, 1, 1.0, [0.2, 0.2], device=dev)
    st.centers = torch.rand((a.H, 2), generator=g, device=dev, dtype=torch.float64)
    st.sigmas = torch.full((a.H, 2), 0.2, dtype=torch.float64, device=dev)
    st.heights = torch.ones((a.H,), dtype=torch.float64, device=dev)
    st.steps = list(range(a.H))
    cv = torch.rand((a.T, 2), generator=g, device=dev, dtype=torch.float64)
    V, dV = st.bias(cv)
    F = torch.empty_like(ds)

    def force():
        _lib.call("mc_mtd_force", _lib.ptr(dV), a.T, 2, _lib.ptr(ds), _lib.ptr(dz), None, _lib.MC_F32, a.N,
                  _lib.ptr(F), _lib.stream_ptr())

    ms = timed(force)
    byt = 3.0 * 12.0 * a.T * a.N
    print(json.dumps({"kernel": "mc_mtd_force", "shape": [a.T, a.N, 3], "ms": ms,
                      "achieved_GBps": byt / ms / 1e6, "peak_GBps": hbm, "frac": byt / ms / 1e6 / hbm}))
    ms = timed(lambda: st.bias(cv, use_grid=False))
    print(json.dumps({"kernel": "mc_mtd_bias_direct", "frames": a.T, "hills": a.H, "ms": ms,
                      "Gexp_per_s": a.T * a.H / ms / 1e6}))
    del ds, dz, F
    toysim_rows(a)


def toysim_rows(a):
    import time

    import numpy as np

    from oracle import toysim as OT
    from paper_1801_02362_b200.toysim import MtdConfig, ToySim, ToySystem, make_references

    sysm = ToySystem(rng_seed=1)
    refs = make_references(sysm, n_refs=16, stride=300)
    for mode in ("close", "original"):
        sim = ToySim(sysm, refs, mode=mode, eps=0.01, mtd=MtdConfig(), walkers=a.W, max_hills=(50 + 3 * a.S) // 50 + 2)
        sim.run(50)
        torch.cuda.synchronize()
        ms = timed(lambda: sim.run(a.S), iters=2)
        sim.check()
        reas = sim.counters[:, 2].double().sum().item()
        steps_done = a.W * (50 + 3 * a.S)
        p = {"bond_k": sysm.bond_k, "bond_r0": sysm.bond_r0, "angle_k": sysm.angle_k, "theta0": sysm.theta0,
             "mob": sysm.mobility, "noise": sysm.noise, "seed": 1, "tau_g": 50, "lam": 100.0, "eps": 0.01,
             "hill_h": 0.5, "hill_sigma": 0.5}
        t0 = time.perf_counter()
        OT.run(p, refs, np.arange(16.0), sysm.initial_chain(), 100, mode=2 if mode == "close" else 1)
        cpu = 100 / (time.perf_counter() - t0)
        print(json.dumps({"kernel": "mc_toysim_run", "mode": mode, "walkers": a.W, "steps": a.S, "beads": 8,
                          "references": 16, "ms": ms, "walker_steps_per_s": a.W * a.S / ms * 1e3,
                          "mean_K": steps_done / max(reas, 1) if mode == "close" else None,
                          "cpu_oracle_steps_per_s_1core": cpu}))


if __name__ == "__main__":
    main()
