"""Per-call timeline of the 20M uniform hull (GPU box diagnostic): host wall
per call, the C side's t_total, and the per-stage CUDA-event times."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1508_05488_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
dist = sys.argv[2] if len(sys.argv) > 2 else "uniform_square"
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate(dist, n, 42, out=h.numpy())
d = h.cuda()
ctx.reserve(n)
torch.cuda.synchronize()
cfg = P.PipelineConfig()
for _ in range(5):
    r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
walls, tots, diags = [], [], []
for _ in range(40):
    t0 = time.perf_counter()
    r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
    walls.append((time.perf_counter() - t0) * 1e3)
    tots.append(r.stats.t_total_ms)
    diags.append(r.diag.times_ms)
out = {"n": n, "dist": dist, "wall_ms_median": float(np.median(walls)), "t_total_median": float(np.median(tots)),
       "stages_median": {k: float(np.median([dd[k] for dd in diags])) for k in diags[0]},
       "launches": r.diag.launches, "kept": sum(r.diag.kept_counts), "cand": r.diag.n_candidates}
# back-to-back loop timed on the host
t0 = time.perf_counter()
for _ in range(40):
    ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
out["loop_ms_per_call"] = (time.perf_counter() - t0) * 1e3 / 40
print(json.dumps(out, indent=1))
