"""Measurement of the §8(f) "next" rows on config-4 shapes (B200):

* neighbour top-M selection (`mc_neighbour_topm`) over a [T, L] fp32 distance
  matrix — HBM-bound: algorithmic bytes = 4 T L read + 4 T M written;
* metadynamics bias force (`mc_mtd_force`) on the path-CV gradients
  [T, N, 3] fp32 (ds, dz) — HBM-bound: 2 x 12 T N read + 12 T N written;
* direct hill sum (`mc_mtd_bias_direct`) for T frames x H hills — one exp per
  (frame, hill): reported as Gexp/s.

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


if __name__ == "__main__":
    main()
