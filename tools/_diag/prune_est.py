"""Diagnostic: fraction of (128-frame tile, 48-landmark tile) pairs that survive
triangle-inequality pruning from a coarse one-term screen (config-4 data)."""
import os, sys, json, math
import torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T, L, N = 16384, 8192, 10000
wl = synth.interp_config_device(4, T, L, N, 32, dev)
lm = torch.from_numpy(wl.landmarks).to(dev)
pcv = engine.PathCVTC(lm, wl.lam, wl.q)
res = {}
for stride in (8, 16, 32):
    coarse = torch.arange(0, L, stride, device=dev)
    C = coarse.numel()
    pc = engine.PathCVTC(lm[coarse].contiguous(), wl.lam)
    Dc, fr, fs = pc.estimate(wl.frames, terms=1)                      # [T, C] one-term estimates
    nx = fs.opnorm
    c_unit = pcv.fcoef / (2 * pcv.lam * pcv.na_max)
    e = c_unit * nx[:, None] * pc.ls.opnorm[None, :]                   # per-pair error bound
    dlo = (Dc.double() - e).clamp_min(0).sqrt()
    dhi = (Dc.double() + e).sqrt()
    dmin_ub = (Dc.double() + e).min(1).values                          # >= true min over all landmarks
    # exact landmark-landmark distances coarse x all
    Dcl = engine.PathCVTC(lm, wl.lam).msd_matrix(lm[coarse].contiguous()).double().clamp_min(0).sqrt()  # [C, L]
    ntl = (L + 47) // 48
    pad = ntl * 48 - L
    Dp = torch.nn.functional.pad(Dcl, (0, pad), value=float("inf"))
    mind = Dp.view(C, ntl, 48).min(2).values                           # [C, ntl]
    # nearest-4 coarse landmarks per frame
    k = 4
    near = Dc.topk(k, dim=1, largest=False).indices                    # [T, k]
    thr = (engine.DEFAULT_CUTOFF + 2.0) / pcv.lam
    lb = torch.zeros((T, ntl), dtype=torch.float64, device=dev)
    for j in range(k):
        c = near[:, j]
        gap = (mind[c] - dhi.gather(1, c[:, None])).clamp_min(0)
        lb = torch.maximum(lb, gap * gap)
    adm = lb <= (dmin_ub[:, None] + thr)                                # admissible (frame, landmark tile)
    # sort frames by nearest coarse landmark, then tile by 128
    order = torch.argsort(near[:, 0] * 1.0 + 0.0)
    a = adm[order]
    ntm = T // 128
    tiles = a.view(ntm, 128, ntl).any(1)
    res[stride] = {"C": C, "frame_adm_frac": float(adm.double().mean()), "tile_frac": float(tiles.double().mean()),
                   "coarse_cost_frac": C / L}
print(json.dumps(res))
