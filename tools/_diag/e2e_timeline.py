"""Timeline of the streamed e2e step (copy stream vs compute stream), config 4."""
import os, sys, json, time
import torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import bench
dev = torch.device("cuda:0")
r = bench.ConfigTC(4, dev, 0, 1)
r.step_device(); torch.cuda.synchronize()
# pure copy of the whole frame set in the same chunks
cps = torch.cuda.Stream(device=dev)
chunks = r.e2e_chunks()
bufs = [torch.empty((n, r.n, 3), dtype=torch.float32, device=dev) for _, n in chunks]
for rep in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cps):
        a.record(cps)
        for (c0, n), buf in zip(chunks, bufs):
            buf.copy_(r.frames_host[c0:c0 + n], non_blocking=True)
        b.record(cps)
    torch.cuda.synchronize()
print(json.dumps({"copy_only_ms": a.elapsed_time(b), "GBps": r.T * r.n * 12 / (a.elapsed_time(b) * 1e6)}))
# compute-only per chunk size (device resident)
comp = []
for (c0, n), buf in zip(chunks, bufs):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(); r._step(buf); b.record(); torch.cuda.synchronize()
    comp.append((n, round(a.elapsed_time(b), 2), round((time.perf_counter() - t0) * 1e3, 2)))
print(json.dumps({"compute_per_chunk": comp, "sum": sum(c[1] for c in comp)}))
# the streamed step with per-chunk events
base = torch.cuda.Event(enable_timing=True)
r.step_e2e(); torch.cuda.synchronize()
evs = []
orig_step = r._step
def stepped(fr, D=None):
    e = torch.cuda.Event(enable_timing=True); e.record()
    out = orig_step(fr, D)
    f = torch.cuda.Event(enable_timing=True); f.record()
    evs.append((e, f))
    return out
r._step = stepped
t0 = time.perf_counter()
base.record()
r.step_e2e()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
print(json.dumps({"e2e_wall_ms": wall, "compute_spans": [(round(base.elapsed_time(e), 1), round(base.elapsed_time(f), 1)) for e, f in evs]}))
