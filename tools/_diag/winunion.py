"""Refine padding under different frame orders: 32-frame groups, 32-landmark sub-tiles."""
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
lo = lo.cpu().numpy().astype(np.int64); cnt = cnt.cpu().numpy().astype(np.int64); hi = lo + cnt
def pad(p, G=32, QL=32):
    a = lo[p].reshape(-1, G).min(1); b = hi[p].reshape(-1, G).max(1)
    u = b - a
    ex = np.ceil(u / QL) * QL
    return {"union": float(u.mean()), "exec_per_frame": float(ex.mean()), "padding": float(ex.mean() / cnt.mean())}
res = {"cnt_mean": float(cnt.mean()), "cnt_p10": float(np.percentile(cnt, 10)), "cnt_p90": float(np.percentile(cnt, 90)),
       "lo": pad(np.argsort(lo, kind="stable")), "mid": pad(np.argsort(lo + hi, kind="stable")),
       "lo_hi": pad(np.lexsort((hi, lo))), "mid_G16": pad(np.argsort(lo + hi, kind="stable"), 16),
       "mid_QL16": pad(np.argsort(lo + hi, kind="stable"), 32, 16), "lo_QL16": pad(np.argsort(lo, kind="stable"), 32, 16)}
print(json.dumps(res))
