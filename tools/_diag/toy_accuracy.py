"""Toy MD: close-structure s vs exact s on the same trajectory, and close vs original runs."""
import numpy as np
import torch

from paper_1801_02362_b200 import engine
from paper_1801_02362_b200.toysim import MtdConfig, ToySim, ToySystem, make_references

for eps in (0.01, 0.003):
    sysm = ToySystem(rng_seed=21)
    refs = make_references(sysm, n_refs=16, stride=300)
    dev = torch.device("cuda:0")
    res = {}
    for mode in ("close", "original"):
        sim = ToySim(sysm, refs, mode=mode, eps=eps, mtd=MtdConfig(), max_hills=200)
        out = sim.run(5000, traj_stride=1)
        sim.check()
        s = out["cv"][0, :, 0].cpu().numpy()
        pcv = engine.PathCV(torch.from_numpy(refs).to(dev), 100.0)
        sx = pcv.evaluate(out["traj"][0], grad=False)["s"].cpu().numpy()
        res[mode] = s
        d = s - sx
        print(f"eps {eps} {mode}: reassign {int(sim.counters[0, 2])} s range [{s.min():.3f}, {s.max():.3f}] "
              f"mean|d| {np.abs(d).mean():.2e} max|d| {np.abs(d).max():.2e} pearson {np.corrcoef(s, sx)[0, 1]:.5f}")
    a, b = res["close"], res["original"]
    lo, hi = min(a.min(), b.min()), max(a.max(), b.max())
    for bins in (50, 20):
        h1, _ = np.histogram(a, bins=bins, range=(lo, hi))
        h2, _ = np.histogram(b, bins=bins, range=(lo, hi))
        print(f"  close vs original runs: hist L1 ({bins} bins) {np.abs(h1 / h1.sum() - h2 / h2.sum()).sum():.3f}")
