import torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
from paper_1801_02362_b200 import engine, synth
dev = torch.device("cuda:0")
wl = synth.walkers_device(3, 4, 10, 2500, 64, dev)
pcv = engine.PathCV(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
print("lraw", pcv.lraw is None, pcv.wuni, engine.CLOSE_DMMA, pcv.n, pcv.w[:3], wl.landmarks.dtype)
wl = synth.walkers_device(3, 256, 1000, 2500, 2048, dev, 0, 16)
pcv = engine.PathCV(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
out = pcv.close_replay(wl.frames, wl.eps, grad=False)
ns = out["nsig"].float()
print("nsig mean", float(ns.mean()), "max", float(ns.max()), "p90", float(ns.quantile(0.9)), "lam", wl.lam)
