"""Group-union padding of the gradient pass under different frame orders (config 4)."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = int(os.environ.get("T", "131072"))
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
Dest, fr, fs, fs0, rlo, rhi, perm0 = pcv._pruned_estimate(wl.frames)
cap = pcv.window_cap
lo, cnt, _, _ = K.candidates(Dest, pcv.lam, pcv.cutoff + pcv.margin, cap, fnorm=pcv.frame_bound(fs), fcoef=2.0 * pcv.lam, rlo=rlo, rhi=rhi)
perm = K.sort_by_key(lo, pcv.L)
Dex, Rex, _ = K.refine(fr, fs, pcv.lraw, pcv.ls, pcv.w, perm=perm, lo=lo, cnt=cnt, cap=cap, fmap=perm0, wuni=pcv.wuni)
wres = K.pathcv_weights(Dex, pcv.q, pcv.lam, Rex, fs, pcv.ls, cap, pcv.cutoff, L=pcv.L, rowlo=lo, rowcnt=cnt)
ns = wres["nsig"].cpu().numpy()
si = wres["sig_idx"].cpu().numpy()
slo = si[np.arange(T), 0]
shi = si[np.arange(T), np.maximum(ns - 1, 0)] + 1
def union(p, G=8):
    a = slo[p].reshape(-1, G).min(1); b = shi[p].reshape(-1, G).max(1)
    return float((b - a).mean())
p_cur = perm.cpu().numpy()
res = {"nsig_mean": float(ns.mean()), "span_mean": float((shi - slo).mean()), "cnt_mean": float(cnt.float().mean()),
       "union_cur": union(p_cur), "union_siglo": union(np.argsort(slo, kind="stable")),
       "union_siglo_hi": union(np.lexsort((shi, slo))), "union_mid": union(np.argsort(slo + shi, kind="stable")),
       "union_cur16": union(p_cur, 16), "union_siglo_hi16": union(np.lexsort((shi, slo)), 16)}
print(json.dumps(res))
