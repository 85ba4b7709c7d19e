"""Metric-pruning statistics (config 4): per-frame hull width vs band union, and the
hulls an exact coarse distance would give."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K, synth
dev = torch.device("cuda:0")
T = int(os.environ.get("T", "131072"))
wl = synth.interp_config_device(4, T, 8192, 10000, 32, dev)
pcv = engine.PathCVTC(torch.from_numpy(wl.landmarks).to(dev), wl.lam, wl.q)
fr0, fs0 = pcv._frames(wl.frames, 1, check=False)
Dc = K.msd_estimate(fs0, pcv.ls_coarse)
ntl = pcv.mind.shape[1]
res = {"lam": pcv.lam, "ntl": ntl, "C": int(pcv.coarse.numel())}
e_tc = (pcv.c_unit * fs0.opnorm[:, None] * pcv.ls_coarse.opnorm[None, :])
res["e_tc_mean"] = float(e_tc.mean()); res["Dc_min_mean"] = float(Dc.min(1).values.mean())
res["window_D_width"] = (pcv.cutoff + 2) / pcv.lam
def stats(Dcx, cunit, knear, tag):
    hlo, hhi, key = K.prune_plan(Dcx, fs0.opnorm, pcv.ls_coarse.opnorm, cunit, pcv.mind, (pcv.cutoff + 2.0) / pcv.lam, knear)
    perm0 = K.sort_by_key(key, ntl + 1)
    tlist, nlist, rlo, rhi = K.band_tiles(perm0, hlo, hhi, 128, 48, pcv.L, ntl)
    w = (hhi - hlo).float()
    res[tag] = {"hull_mean": float(w.mean()), "hull_p90": float(w.quantile(0.9)), "frac": int(nlist.item()) / (((T + 127) // 128) * ntl)}
stats(Dc, pcv.c_unit, 4, "onet_k4")
stats(Dc, pcv.c_unit, 8, "onet_k8")
# split (3-term) coarse estimate with its measured margin folded in as the error term
fs3 = K.center_split(fr0, pcv.wa, pcv.w, weighted=False, fmt=pcv.fmt, terms=3)
lc3 = K.center_split(pcv.lraw[pcv.coarse].contiguous(), pcv.wa, pcv.w, weighted=True, moments=False, fmt=pcv.fmt, terms=3)
Dc3 = K.msd_estimate(fs3, lc3)
res["err3_vs_1_max"] = float((Dc3 - Dc).abs().max())
stats(Dc3, 1e-9, 4, "split3_k4_tinyerr")
stats(Dc3, 1e-9, 8, "split3_k8_tinyerr")
print(json.dumps(res))
