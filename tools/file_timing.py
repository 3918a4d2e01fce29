"""Time chgpu_hull_xy_binary (file in page cache) vs chgpu_hull from a numpy
array vs from pinned memory, 20M uniform."""
import os, sys, time, tempfile
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1508_05488_b200 as P
ctx = P.Context(0)
pts = P.generate("uniform_square", 20_000_000, 42)
f = os.path.join(tempfile.gettempdir(), "u20m.xyb")
np.ascontiguousarray(pts, dtype="<f8").tofile(f)
pin = torch.empty((len(pts), 2), dtype=torch.float64, pin_memory=True); pin.numpy()[:] = pts
def t(fn, k=10):
    for _ in range(3): fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); r = fn(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3, r
ms, r = t(lambda: ctx.hull_xy_binary(f, copy=False))
print("file (page cache) %.2f ms  h2d %.2f" % (ms, r.diag.times_ms["t_h2d_ms"]))
ms, r = t(lambda: ctx.convex_hull(pts, copy=False))
print("pageable numpy   %.2f ms  h2d %.2f" % (ms, r.diag.times_ms["t_h2d_ms"]))
ms, r = t(lambda: ctx.convex_hull(pin.numpy(), copy=False))
print("pinned           %.2f ms  h2d %.2f" % (ms, r.diag.times_ms["t_h2d_ms"]))
t0 = time.perf_counter(); a = np.fromfile(f, dtype="<f8"); t1 = time.perf_counter()
print("np.fromfile alone %.2f ms" % ((t1 - t0) * 1e3))
os.remove(f)
