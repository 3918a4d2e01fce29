"""K1+K2 in-step with and without the programmatic launch of K2."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
n = 20_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
cfg = P.PipelineConfig()
for pdl in (False, True, False, True):
    ctx.set_pdl(pdl)
    for _ in range(5): ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
    k12, tot, wall = [], [], []
    for _ in range(30):
        t0 = time.perf_counter()
        r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
        wall.append((time.perf_counter() - t0) * 1e3)
        t = r.diag.times_ms
        k12.append(t["t_k1_ms"] + t["t_k2_ms"]); tot.append(r.stats.t_total_ms)
    print(f"pdl={pdl} k1+k2 {np.median(k12)*1e3:.1f} us  total {np.median(tot)*1e3:.1f} us wall {np.median(wall)*1e3:.1f} us  hull {r.stats.n_hull} spa {r.stats.n_after_spa}")
