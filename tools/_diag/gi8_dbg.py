"""Diagnostic: one small mc_pathcv_grad_i8 call (MC_GI8_DBG selects stages to skip)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1801_02362_b200 import engine, synth
wl = synth.config4(seed=5, T=int(os.environ.get("T", 16)), L=256, N=int(os.environ.get("N", 512)))
pcv = engine.PathCVTC(wl.landmarks, wl.lam)
out = pcv.evaluate(wl.frames)
torch.cuda.synchronize()
print("ok", os.environ.get("MC_GI8_DBG"), float(out["ds"].abs().max()))
