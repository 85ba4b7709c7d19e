"""Micro-benchmark of the tcgen05 3xTF32 covariance + MSD-estimate kernel.

    python tools/perf_tf32.py --T 16384 --L 8192 --n 10000 [--iters 3]

Prints kernel time (CUDA events), executed TF32 TFLOP/s (3 x 18 n per pair)
and the estimate error statistics on a subsample checked against the exact
fp64 device path.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))

from paper_1801_02362_b200 import engine, kernels as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--L", type=int, default=8192)
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--check", type=int, default=64, help="frames checked against the exact path")
    ap.add_argument("--fmt", default="f16", choices=["f16", "tf32"])
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    T, L, n = args.T, args.L, args.n
    lm = (torch.randn((L, n, 3), generator=g, device=dev) * 0.3).float()
    base = lm[torch.randint(0, L, (T,), generator=g, device=dev)]
    sig = torch.exp(torch.empty(T, device=dev).uniform_(np.log(1e-3), np.log(0.5), generator=g))
    fr = (base + torch.randn((T, n, 3), generator=g, device=dev) * sig[:, None, None]).float()
    w = engine.normalise_weights(None, n, "d", dev)
    fs = K.center_split(fr, w, w, weighted=False, fmt=args.fmt)
    ls = K.center_split(lm, w, w, weighted=True, fmt=args.fmt)
    D = torch.empty((T, L), dtype=torch.float32, device=dev)
    K.msd_tf32(fs, ls, D)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        K.msd_tf32(fs, ls, D)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    flop = 3.0 * 18.0 * n * T * L
    out = {"fmt": args.fmt, "two_sm": K.TF32_2SM, "T": T, "L": L, "n": n, "ms": ms, "tflops_executed": flop / ms / 1e9,
           "useful_tflops": flop / 3 / ms / 1e9, "pairs_per_s": T * L / ms * 1e3}
    if args.check:
        c = args.check
        pcv = engine.PathCV(lm, 1.0)
        ex = pcv.msd_matrix(fr[:c]).cpu().numpy()
        est = D[:c].double().cpu().numpy()
        err = np.abs(est - ex)
        out.update(err_max=float(err.max()), err_median=float(np.median(err)),
                   err_p99=float(np.quantile(err, 0.99)), rel_err_max=float((err / np.maximum(ex, 1e-12)).max()))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
