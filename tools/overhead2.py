"""Per-call overhead outside the C-side wall clock: Python loop time per
call vs StageStats.t_total_ms, 20M uniform device-resident."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
import paper_1508_05488_b200 as P
ctx = P.Context(0)
pts = P.generate("uniform_square", 20_000_000, 42)
d = torch.from_numpy(pts).cuda(); torch.cuda.synchronize()
cfg = P.PipelineConfig()
for _ in range(5): ctx.convex_hull_device(d.data_ptr(), len(pts), cfg, copy=False)
N = 50
walls = []
t0 = time.perf_counter()
for _ in range(N):
    r = ctx.convex_hull_device(d.data_ptr(), len(pts), cfg, copy=False)
    walls.append(r.stats.t_total_ms)
t1 = time.perf_counter()
print(f"python per call {(t1 - t0) / N * 1e3:.4f} ms, C wall median {np.median(walls):.4f} ms")
