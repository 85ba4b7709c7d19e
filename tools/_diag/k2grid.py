"""Pipeline K2 -> refine -> grad timing vs the screening GEMM's CTA count (power cap)."""
import os, sys, json, time
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = 131072
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
res = {}
grids = [int(g) for g in os.environ.get("GRIDS", "0,136,124,112,100").split(",")]
for g in grids:
    engine.K2_GRID = g
    for _ in range(2):
        pcv.evaluate(wl.frames)
    torch.cuda.synchronize()
    time.sleep(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4):
        pcv.evaluate(wl.frames)
    b.record(); torch.cuda.synchronize()
    res[g] = round(a.elapsed_time(b) / 4, 1)
print(json.dumps(res))
