import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = 16384
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
fr = wl.frames
Dest, frc, fs = pcv.estimate(fr)
lo, cnt, _, _ = K.candidates(Dest, pcv.lam, pcv.cutoff + pcv.margin, pcv.window_cap)
perm = K.sort_by_key(lo, pcv.L)
out = pcv.evaluate(fr, grad=False)
nsig = out["nsig"].cpu().numpy()
lo_ = lo.cpu().numpy(); cnt_ = cnt.cpu().numpy(); p = perm.cpu().numpy()
# sig lists are not returned; approximate the sig span by the window
lo_p = lo_[p]; hi_p = lo_p + cnt_[p]
G = 8
ng = T // G
u8 = [(hi_p[g*G:(g+1)*G].max() - lo_p[g*G:(g+1)*G].min()) for g in range(ng)]
G32 = 32
u32 = [(hi_p[g*G32:(g+1)*G32].max() - lo_p[g*G32:(g+1)*G32].min()) for g in range(T // G32)]
print(json.dumps({"lam": pcv.lam, "margin": pcv.margin, "cnt_mean": float(cnt_.mean()), "cnt_max": int(cnt_.max()),
                  "nsig_mean": float(nsig.mean()), "nsig_max": int(nsig.max()),
                  "union8_mean": float(np.mean(u8)), "union8_p90": float(np.percentile(u8, 90)), "union8_max": int(np.max(u8)),
                  "union32_mean": float(np.mean(u32)), "union32_max": int(np.max(u32)),
                  "G_frames_mean": float(fs.g.mean().item()), "G_lm_mean": float(pcv.ls.g.mean().item())}))
