import torch, time
n = 390_000_000
h = torch.empty(n, dtype=torch.int32).pin_memory()
print("pinned", h.is_pinned())
d = torch.empty(n, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
for i in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s):
        for c in range(16):
            a, b = c * n // 16, (c + 1) * n // 16
            d[a:b].copy_(h[a:b], non_blocking=True)
    t1 = time.perf_counter()
    s.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e3*(t1-t):.2f} ms total {1e3*(t2-t):.2f} ms  {n*4/(t2-t)/1e9:.1f} GB/s")
