"""Gradient truncation study: ds/dz from significant lists cut at lam (D - Dmin) <= c
vs the c = 25 lists (config 4 generator)."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = int(os.environ.get("T", "32768"))
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
Dest, fr, fs, fs0, rlo, rhi, perm0 = pcv._pruned_estimate(wl.frames)
cap = pcv.window_cap
lo, cnt, _, _ = K.candidates(Dest, pcv.lam, pcv.cutoff + pcv.margin, cap, fnorm=pcv.frame_bound(fs), fcoef=2.0 * pcv.lam, rlo=rlo, rhi=rhi)
perm = K.sort_by_key((2 * lo + cnt).to(torch.int32), 2 * pcv.L + 1)
Dex, Rex, _ = K.refine(fr, fs, pcv.lraw, pcv.ls, pcv.w, perm=perm, lo=lo, cnt=cnt, cap=cap, fmap=perm0, wuni=pcv.wuni)
def grad(cut):
    wres = K.pathcv_weights(Dex, pcv.q, pcv.lam, Rex, fs, pcv.ls, cap, cut, L=pcv.L, rowlo=lo, rowcnt=cnt)
    gperm = K.sort_by_key(K.sig_span_key(wres, pcv.L), 2 * pcv.L + 1)
    ds, dz = K.pathcv_grad_block(wres, fs, pcv.ls, fr, pcv.lraw, pcv.w, pcv.wa, cap, gperm, torch.float64, out_map=perm0)
    return ds, dz, float(wres["nsig"].float().mean())
ds0, dz0, n0 = grad(25.0)
res = {"nsig25": n0}
for c in (20.0, 17.0, 15.0, 13.0, 11.0):
    ds, dz, nm = grad(c)
    r = {"nsig": nm}
    for nm_, a, b in (("ds", ds, ds0), ("dz", dz, dz0)):
        sc = b.abs().reshape(T, -1).amax(1)
        er = (a - b).abs().reshape(T, -1).amax(1) / sc
        r[nm_ + "_max"] = float(er.max()); r[nm_ + "_p99"] = float(er.quantile(0.99)); r[nm_ + "_gt1e6"] = float((er > 1e-6).float().mean())
    res[c] = r
print(json.dumps(res))
