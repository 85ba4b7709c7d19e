import os, sys, json, time
import torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import bench
dev = torch.device("cuda:0")
r = bench.ConfigTC(4, dev, 0, 1)
r.step_device(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); r.step_device(); e1.record(); torch.cuda.synchronize()
print(json.dumps({"device_ms": e0.elapsed_time(e1)}))
for sched in os.environ.get("SCHEDS", "4096,24576,1.5,0;4096,24576,1.5,1;2048,24576,1.5,1;4096,16384,1.5,1;4096,32768,1.5,1;2048,12288,1.5,1").split(";"):
    os.environ["MC_E2E_CHUNKS"] = sched
    r.step_e2e(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); r.step_e2e(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"sched": sched, "chunks": len(r.e2e_chunks()), "e2e_ms": min(ts)}))
