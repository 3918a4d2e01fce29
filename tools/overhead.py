"""Per-call time split: C-side wall time (StageStats.t_total_ms) vs the
Python wrapper call vs CUDA-event step time, 20M uniform device-resident."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1508_05488_b200 as P
ctx = P.Context(0)
pts = P.generate("uniform_square", 20_000_000, 42)
d = torch.from_numpy(pts).cuda(); torch.cuda.synchronize()
cfg = P.PipelineConfig()
for _ in range(5): ctx.convex_hull_device(d.data_ptr(), len(pts), cfg, copy=False)
tt, tc = [], []
for _ in range(20):
    t0 = time.perf_counter(); r = ctx.convex_hull_device(d.data_ptr(), len(pts), cfg, copy=False); t1 = time.perf_counter()
    tt.append((t1 - t0) * 1e3); tc.append(r.stats.t_total_ms)
print("python call %.3f ms  C wall %.3f ms  (median)" % (np.median(tt), np.median(tc)))
print("diag times", {k: round(v, 4) for k, v in r.diag.times_ms.items()})
print("stats", r.stats)
