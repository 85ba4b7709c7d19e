import torch, time, json
dev = torch.device("cuda:0")
res = {}
for mb in (256, 1024):
    h = torch.empty(mb * 2**20 // 4, dtype=torch.float32).pin_memory()
    d = torch.empty_like(h, device=dev)
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    res[f"h2d_{mb}MB_GBps"] = 5 * mb * 2**20 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    # concurrent with a compute-heavy kernel on another stream
    s = torch.cuda.Stream()
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    e0.record()
    with torch.cuda.stream(s):
        for _ in range(5):
            d.copy_(h, non_blocking=True)
    for _ in range(40):
        a @ a
    e1.record(); torch.cuda.synchronize()
    res[f"h2d_{mb}MB_with_gemm_ms"] = e0.elapsed_time(e1)
print(json.dumps(res))
