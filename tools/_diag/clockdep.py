"""Kernel time vs sustained load: refine / grad launched back to back vs after idle."""
import os, sys, json, time, subprocess, threading
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = 131072
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
Dest, fr, fs, fs0, rlo, rhi, perm0 = pcv._pruned_estimate(wl.frames)
cap = pcv.window_cap
lo, cnt, _, _ = K.candidates(Dest, pcv.lam, pcv.cutoff + pcv.margin, cap, fnorm=pcv.frame_bound(fs), fcoef=2.0 * pcv.lam, rlo=rlo, rhi=rhi)
perm = K.sort_by_key((2 * lo + cnt).to(torch.int32), 2 * pcv.L + 1)
def rf():
    return K.refine(fr, fs, pcv.lraw, pcv.ls, pcv.w, perm=perm, lo=lo, cnt=cnt, cap=cap, fmap=perm0, wuni=pcv.wuni)
Dex, Rex, _ = rf()
wres = K.pathcv_weights(Dex, pcv.q, pcv.lam, Rex, fs, pcv.ls, cap, pcv.cutoff, L=pcv.L, rowlo=lo, rowcnt=cnt)
gperm = K.sort_by_key(K.sig_span_key(wres, pcv.L), 2 * pcv.L + 1)
def gr():
    return K.pathcv_grad_block(wres, fs, pcv.ls, fr, pcv.lraw, pcv.w, pcv.wa, cap, gperm, torch.float32, out_map=perm0)
def k2():
    return pcv._pruned_estimate(wl.frames)
smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=timestamp,clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "50"], stdout=open("gpurun_out/clk.csv", "w"))
def t1(fn, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return ts
res = {}
for name, fn in (("refine", rf), ("grad", gr), ("k2", k2)):
    time.sleep(2.0)
    res[name + "_cold"] = t1(fn, 1)
    res[name + "_hot"] = t1(fn, 8)
    # back to back without host sync between launches
    time.sleep(2.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(8): fn()
    b.record(); torch.cuda.synchronize()
    res[name + "_b2b_avg"] = a.elapsed_time(b) / 8
# pipeline order: K2 -> refine -> grad, each timed on the stream
time.sleep(2.0)
seq = []
for _ in range(6):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(); k2(); ev[1].record(); rf(); ev[2].record(); gr(); ev[3].record()
    seq.append(ev)
torch.cuda.synchronize()
res["pipe_k2"] = [e[0].elapsed_time(e[1]) for e in seq]
res["pipe_refine"] = [e[1].elapsed_time(e[2]) for e in seq]
res["pipe_grad"] = [e[2].elapsed_time(e[3]) for e in seq]
# refine after an idle gap following K2
seq = []
for _ in range(4):
    k2(); torch.cuda.synchronize(); time.sleep(0.5)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); rf(); b.record(); torch.cuda.synchronize(); seq.append(a.elapsed_time(b))
res["refine_after_k2_gap"] = seq
smi.terminate()
print(json.dumps({k: (np.round(v, 1).tolist() if isinstance(v, list) else round(v, 1)) for k, v in res.items()}))
