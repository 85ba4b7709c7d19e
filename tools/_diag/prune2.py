"""Prototype of the two-sided triangle bound for the metric pruning (torch on GPU):
LB1 = (mind[c,tau] - dhi(t,c))^2 over the knear nearest coarse landmarks (current),
LB2 = (dlo(t,c) - maxd[c,tau])^2 over the coarse landmarks inside / next to tau."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = int(os.environ.get("T", "32768"))
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q, coarse_stride=int(os.environ.get("STRIDE", "16")))
fr0, fs0 = pcv._frames(wl.frames, 1, check=False)
Dc = K.msd_estimate(fs0, pcv.ls_coarse).double()
C = Dc.shape[1]; L = pcv.L; ntl = (L + 47) // 48
e = pcv.c_unit * fs0.opnorm.double()[:, None] * pcv.ls_coarse.opnorm.double()[None, :]
dhi = (Dc + e).clamp_min(0).sqrt(); dlo = (Dc - e).clamp_min(0).sqrt()
dub = (Dc + e).min(1).values
lim = dub + (pcv.cutoff + 2.0) / pcv.lam
# exact coarse -> landmark distances
lc = pcv.lraw[pcv.coarse].contiguous()
dcl = torch.empty((C, L), dtype=torch.float32, device=dev)
fsc = K.center_split(lc, pcv.wa, pcv.w, weighted=False, fmt=pcv.fmt)
K.refine(lc, fsc, pcv.lraw, pcv.ls, pcv.w, Dd=dcl)
rm = dcl.double().clamp_min(0).sqrt()
rmp = torch.nn.functional.pad(rm, (0, ntl * 48 - L), value=float("nan"))
v = rmp.view(C, ntl, 48)
mind = torch.nan_to_num(v, nan=float("inf")).amin(2) * (1 - 1e-6)
maxd = torch.nan_to_num(v, nan=0.0).amax(2) * (1 + 1e-6) + 1e-7
# LB1 (current: knear nearest coarse by estimate)
kn = 4
near = Dc.topk(kn, dim=1, largest=False).indices             # [T, kn]
lb1 = torch.zeros((T, ntl), dtype=torch.float64, device=dev)
for k in range(kn):
    c = near[:, k]
    g = (mind[c] - dhi.gather(1, c[:, None])).clamp_min(0)
    lb1 = torch.maximum(lb1, g * g)
# LB2: coarse landmarks c with index in [tau*48 - 48, tau*48 + 96) (own tile +- one tile)
stride = L // C
lb2 = torch.zeros((T, ntl), dtype=torch.float64, device=dev)
tau = torch.arange(ntl, device=dev)
span = 48 // stride + 1
for off in range(-span, 2 * span + 1):
    cidx = (tau * 48) // stride + off
    ok = (cidx >= 0) & (cidx < C)
    cc = cidx.clamp(0, C - 1)
    g = (dlo[:, cc] - maxd[cc, tau][None, :]).clamp_min(0)
    g = torch.where(ok[None, :], g, torch.zeros_like(g))
    lb2 = torch.maximum(lb2, g * g)
def frac(lb):
    adm = lb <= lim[:, None]
    lo = torch.where(adm, tau[None, :], ntl).amin(1); hi = torch.where(adm, tau[None, :], -1).amax(1) + 1
    return float((hi - lo).float().mean()), float(adm.float().sum(1).mean()), lo, hi
r = {}
for name, lb in (("lb1", lb1), ("lb2", lb2), ("max", torch.maximum(lb1, lb2))):
    hm, am, lo, hi = frac(lb)
    key = torch.where(hi - lo >= (3 * ntl) // 4, 0, 1 + lo).int()
    perm = K.sort_by_key(key.contiguous(), ntl + 1)
    tl, nl, _, _ = K.band_tiles(perm, lo.int().contiguous(), hi.int().contiguous(), 128, 48, L, ntl)
    r[name] = {"hull_mean": hm, "admissible_mean": am, "band_frac": int(nl.item()) / (((T + 127) // 128) * ntl)}
r["Dmin_mean"] = float(Dc.min(1).values.mean()); r["maxd_mean"] = float(maxd[torch.arange(C), (torch.arange(C) * stride) // 48].mean())
print(json.dumps(r))
