"""H2D bandwidth from pinned host memory: one stream vs two / four concurrent streams."""
import torch

dev = torch.device("cuda:0")
nbytes = 4 << 30
h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
d = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        parts = h.chunk(ns * 8)
        dparts = d.chunk(ns * 8)
        for i, (a, b) in enumerate(zip(parts, dparts)):
            s = streams[i % ns]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                b.copy_(a, non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(f"{ns} stream(s): {nbytes / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
