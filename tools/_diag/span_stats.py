"""Config-4 significant-span statistics: per-frame span (last - first + 1) and the
8-frame group union widths under the grouping key first + last and under a
width-bucketed key.  Diagnostic."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1801_02362_b200 import engine, kernels as K, synth

T = int(os.environ.get("T", 32768))
L, N = 8192, 10000
dev = torch.device("cuda:0")
wl = synth.interp_config_device(4, T, L, N, 32, dev)
pcv = engine.PathCVTC(wl.landmarks, wl.lam)
cap = {}
orig = K.pathcv_grad_block
def grab(wres, *a, **k):
    cap["idx"] = wres["sig_idx"].clone(); cap["ns"] = wres["nsig"].clone()
    return orig(wres, *a, **k)
K.pathcv_grad_block = grab
pcv.evaluate(wl.frames)
idx, ns = cap["idx"], cap["ns"].long()
first = idx[:, 0].long(); last = idx.gather(1, (ns - 1).clamp_min(0)[:, None])[:, 0].long()
span = (last - first + 1).cpu().numpy(); nsn = ns.cpu().numpy()
print("T", T, "nsig mean %.1f p50 %d p90 %d p99 %d max %d" % (nsn.mean(), np.median(nsn), np.percentile(nsn, 90), np.percentile(nsn, 99), nsn.max()))
print("span mean %.1f p50 %d p90 %d p99 %d max %d" % (span.mean(), np.median(span), np.percentile(span, 90), np.percentile(span, 99), span.max()))
f, l_ = first.cpu().numpy(), last.cpu().numpy()
def groups(order, G=8):
    o = order[: (len(order) // G) * G].reshape(-1, G)
    w = l_[o].max(1) - f[o].min(1) + 1
    return w
for name, key in (("first+last", f + l_), ("width-bucket", (np.minimum(span, 200) // 8) * (2 * L + 1) + f + l_)):
    for G in (8, 16):
        w = groups(np.argsort(key, kind="stable"), G)
        print(f"{name:13s} G={G:2d}: union mean {w.mean():.1f} p90 {np.percentile(w, 90):.0f} p99 {np.percentile(w, 99):.0f} "
              f"> 80: {100 * (w > 80).mean():.1f}%  > 120: {100 * (w > 120).mean():.1f}%  sum(3w)/sum(3 span) {w.sum() * G / span.sum():.3f}")
