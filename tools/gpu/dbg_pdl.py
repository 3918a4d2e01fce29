import sys; sys.path.insert(0, ".")
import numpy as np, paper_1508_05488_b200 as P
ctx = P.Context(0)
pts = P.generate("uniform_disk", 20_000_000, 3)
for pdl in (False, True, True, False, True):
    ctx.set_pdl(pdl)
    for cc in (1, 1024):
        r = ctx.convex_hull(pts, P.PipelineConfig(chunk_count=cc))
        print(pdl, cc, r.diag.region_counts, r.stats.n_hull, r.diag.quad.ravel()[:4], r.diag.k1k2_overlapped)
import torch
d = torch.from_numpy(pts).cuda(); torch.cuda.synchronize()
for pdl in (False, True):
    ctx.set_pdl(pdl)
    r = ctx.convex_hull_device(d.data_ptr(), len(pts), P.PipelineConfig(chunk_count=1))
    print("dev", pdl, r.diag.region_counts, r.stats.n_hull)
