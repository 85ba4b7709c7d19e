import os, sys, json
import torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = int(os.environ.get("T", "32768"))
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
fr = wl.frames
_, fs = pcv._frames(fr, 1)
D = torch.empty((T, 8192), dtype=torch.float32, device=dev)
K.msd_estimate(fs, pcv.ls, D); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    K.msd_estimate(fs, pcv.ls, D)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"lib": os.environ.get("MCB200_LIB", "default"), "T": T, "ms": e0.elapsed_time(e1) / 3}))
