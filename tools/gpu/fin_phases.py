"""A few hulls of N uniform points (seed 42), device-resident: run under a
library built with -DCHGPU_FINISH_CLOCKS=1 (CHGPU_LIB) to print k_spa_finish's
phase clocks. usage: fin_phases.py N"""
import sys, torch
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
n = int(sys.argv[1])
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
for _ in range(3):
    r = ctx.convex_hull_device(d.data_ptr(), n, P.PipelineConfig(), copy=False)
    torch.cuda.synchronize()
print(r.stats.n_hull, r.diag.n_candidates)
