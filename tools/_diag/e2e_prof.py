import os, sys, json, time
import torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import bench
from paper_1801_02362_b200 import _lib
dev = torch.device("cuda:0")
r = bench.ConfigTC(4, dev, 0, 1)
r.step_e2e(); torch.cuda.synchronize()
for chunk in (16384, 32768, 65536):
    r.chunk = chunk
    r.step_e2e(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.start_profile()
    r.step_e2e()
    prof = _lib.stop_profile()
    wall = (time.perf_counter() - t0) * 1e3
    tot = sum(t for _, t in prof.values())
    t0 = time.perf_counter(); r.step_e2e(); torch.cuda.synchronize(); wall2 = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"chunk": chunk, "wall_ms_profiled": wall, "wall_ms": wall2, "kernel_sum_ms": tot,
                      "kernels": {k: round(v[1], 1) for k, v in prof.items()}}))
