"""D2H bandwidth of a 320 MB copy into pinned memory: one copy, or split
across two streams."""
import time, torch
n = 320 * 1024 * 1024 // 8
d = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("one", "two", "one", "two", "four"):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if mode == "one":
            with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
        else:
            k = 2 if mode == "two" else 4
            ss = [s1, s2] if k == 2 else [torch.cuda.Stream() for _ in range(4)]
            step = n // k
            for i in range(k):
                with torch.cuda.stream(ss[i % len(ss)]): h[i*step:(i+1)*step].copy_(d[i*step:(i+1)*step], non_blocking=True)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(mode, f"{min(ts)*1e3:.2f} ms  {n*8/min(ts)/1e9:.1f} GB/s")
