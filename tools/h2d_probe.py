import torch, time
n = 320_000_000
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for chunk in (n, 64 << 20, 32 << 20, 16 << 20, 8 << 20):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for off in range(0, n, chunk):
                d[off:off+chunk].copy_(h[off:off+chunk], non_blocking=True)
            e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"chunk {chunk>>20:4d} MB: {best:.3f} ms  {n/best/1e6:.1f} GB/s")

# two copy streams alternating chunks (both copy engines, if the driver uses them)
s2 = torch.cuda.Stream()
for chunk in (32 << 20, 64 << 20):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        s2.wait_event(e0)
        for i, off in enumerate(range(0, n, chunk)):
            st = s if i % 2 == 0 else s2
            with torch.cuda.stream(st):
                d[off:off+chunk].copy_(h[off:off+chunk], non_blocking=True)
        s.wait_stream(s2)
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"2 streams, chunk {chunk>>20:4d} MB: {best:.3f} ms  {n/best/1e6:.1f} GB/s")
