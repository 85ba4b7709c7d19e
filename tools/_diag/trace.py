import os, sys, json, time
import numpy as np, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1801_02362_b200 import engine, kernels as K
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
T, L, n = 16384, 8192, 10000
lm = (torch.randn((L, n, 3), generator=g, device=dev) * 0.3).float()
fr = (lm[torch.randint(0, L, (T,), generator=g, device=dev)] + 0.01 * torch.randn((T, n, 3), generator=g, device=dev)).float()
w = engine.normalise_weights(None, n, "d", dev)
fs = K.center_split(fr, w, w, weighted=False, fmt="f16")
ls = K.center_split(lm, w, w, weighted=True, fmt="f16")
Dx = torch.zeros((T + 8, L), dtype=torch.float32, device=dev)
D = Dx[:T]
K.msd_estimate(fs, ls, D, two_sm=False)
torch.cuda.synchronize()
Dx.zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
K.msd_estimate(fs, ls, D, two_sm=False)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"kernel_ms": e0.elapsed_time(e1)}))
flat = Dx[T:].contiguous().view(torch.int64).flatten()
tr = flat[: 4 * 313].view(313, 4).cpu().numpy()
te = flat[4 * 4096: 4 * 4096 + 2 * 148].view(148, 2).cpu().numpy()
te = te[te[:, 0] != 0]
gaps = te[1:, 0] - te[:-1, 0]
tw = te[:, 1] - te[:, 0]
ep = flat[5 * 4096: 5 * 4096 + 16 * 148].view(148, 8, 2).cpu().numpy()
ep = ep[ep[:, 0, 0] != 0]
dur = ep[:, :, 1] - ep[:, :, 0]
print(json.dumps({"epi_warp_dur_p50": float(np.median(dur)), "epi_warp_dur_max_p50": float(np.median(dur.max(1))),
                  "epi_start_spread_p50": float(np.median(ep[:, :, 0].max(1) - ep[:, :, 0].min(1))),
                  "last_commit_to_epi_start_p50": float(np.median(ep[1:, :, 0].min(1) - te[1:len(ep), 0])) if len(ep) > 1 else None}))
mt = flat[6 * 4096: 6 * 4096 + 8 * 148].view(148, 8).cpu().numpy()
print(json.dumps({"math_cycles_chunk_p50": [float(np.median(mt[1:, c])) for c in (0, 2, 4)]}))
print(json.dumps({"tiles": len(te), "tile_period_p50": float(np.median(gaps)), "tempty_wait_p50": float(np.median(tw)),
                  "tempty_wait_mean": float(tw[1:].mean()), "tile_period_mean": float(gaps.mean())}))
t0 = tr[:, 0].min()
tr = tr - t0
pw = tr[:, 1] - tr[:, 0]
mw = tr[:, 3] - tr[:, 2]
span = tr[-1, 3] - tr[0, 2]
print(json.dumps({"stages": 313, "span_cycles": int(span), "cycles_per_stage": float(span / 312),
                  "mma_full_wait_total": int(mw[1:].sum()), "mma_full_wait_frac": float(mw[1:].sum() / span),
                  "mma_wait_p50": float(np.median(mw)), "mma_wait_max": int(mw.max()),
                  "prod_empty_wait_p50": float(np.median(pw)),
                  "mma_iter_gap_p50": float(np.median(np.diff(tr[:, 2]))),
                  "first": tr[:8].tolist()}))
